"""End-to-end Anderson-accelerated FWI on the GPU (BASELINE C3: AA m=10,
30 iterations, fp32), device-resident optimizer loop.

    python tools/run_inversion.py [--config c3] [--iters 30] [--memory 10] [--csv out.csv]

Prints per-iteration rows (objective, |g|, evaluation counters, lambda) and
the wall time; the model error |m - m_true| / |m_true| at the start and end."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--memory", type=int, default=10)
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2008_11778_b200 import anderson, gradients, synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case(a.config)
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    prop = Propagator(grid, geom, wav, cfg, dtype="float32")
    prop.set_model(case["true"].m)
    obs = prop.synthetic()
    prop.close()
    obj = gradients.FwiObjective(grid, obs, wav, geom, cfg, dtype="float32")
    m_true = torch.as_tensor(case["true"].m.ravel(), device="cuda", dtype=torch.float32)
    p0 = torch.as_tensor(case["init"].m.ravel(), device="cuda", dtype=torch.float32)
    err0 = float((p0 - m_true).norm() / m_true.norm())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = anderson.minimize_aa(obj, p0, memory=a.memory, max_iters=a.iters)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    err1 = float((res.p - m_true).norm() / m_true.norm())
    print("iter objective grad_norm grad_evals obj_evals lambda")
    for r in res.report.rows:
        print(f"{r.iteration:4d} {r.objective:.6e} {r.grad_norm:.4e} {r.grad_evals:4d} "
              f"{r.obj_evals:4d} {r.step:.4g}")
    rows = res.report.rows
    print(f"{a.config}: {a.iters} AA(m={a.memory}) iterations in {wall:.2f} s "
          f"({rows[-1].grad_evals} gradients + {rows[-1].obj_evals} misfit evaluations); "
          f"objective {rows[0].objective:.4e} -> {rows[-1].objective:.4e} "
          f"({rows[-1].objective / rows[0].objective:.3f}); model error {err0:.4e} -> {err1:.4e}")
    if a.csv:
        res.report.to_csv(a.csv)


if __name__ == "__main__":
    main()

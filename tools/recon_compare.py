"""Gradient time by reconstruction mode (CUDA events, one GPU).

    python tools/recon_compare.py --config c3 --modes full,boundary [--reps 3]

For every mode: warm-up gradient, then `reps` timed gradients; plus the step
kernels of the mode timed in isolation (forward/adjoint, or for boundary the
band-saving forward and the fused reverse+adjoint step)."""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--modes", default="full,boundary")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--budget", type=float, default=0.0, help="device memory budget, GB")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case(a.config, n_shots=a.shots or None)
    geom = case["geometry"]
    S = geom.n_sources
    obs = torch.zeros((S, geom.nt, geom.n_receivers), device="cuda", dtype=torch.float32)
    for mode in a.modes.split(","):
        prop = Propagator(case["grid"], geom, case["wavelet"], case["config"], dtype="float32",
                          recon=mode, mem_budget_bytes=a.budget * 1e9)
        prop.set_model(case["init"].m)
        # observed data = synthetic of the true model (first call also warms up)
        if mode == a.modes.split(",")[0]:
            prop.set_model(case["true"].m)
            obs = prop.synthetic()
            prop.set_model(case["init"].m)
        t0 = time.time()
        v, g = prop.gradient(obs)
        torch.cuda.synchronize()
        warm = time.time() - t0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            v, g = prop.gradient(obs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        q = prop.query()
        if mode == "boundary":
            kf = prop.time_step_kernel(6, q["batch"], 20)
            kb = prop.time_step_kernel(5, q["batch"], 20)
        else:
            kf = prop.time_step_kernel(0, q["batch"], 20) if mode == "full" else float("nan")
            kb = prop.time_step_kernel(1, q["batch"], 20) if mode == "full" else float("nan")
        gn = float(g.double().norm())
        print(f"{a.config} {mode}: {ms:.1f} ms/gradient (first {warm:.1f} s), batch {q['batch']}, "
              f"{q['device_bytes'] / 1e9:.1f} GB, misfit {v:.6e}, |g| {gn:.6e}, "
              f"fwd step {kf * 1e3:.1f} us, adj step {kb * 1e3:.1f} us", flush=True)
        if mode == a.modes.split(",")[0]:
            g_ref = g.clone()
        else:
            print(f"   rel diff vs {a.modes.split(',')[0]}: "
                  f"{float((g - g_ref).double().norm() / g_ref.double().norm()):.3e}")
        del prop
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

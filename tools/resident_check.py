"""A/B of the cluster-resident whole-sweep kernels against the one-step
kernels on one config: results (bitwise / relative) and device time.

    python tools/resident_check.py [--config c3] [--shots N] [--nt N] [--reps 3]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--shots", type=int, default=None)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    if a.config == "c1":
        case = synthetic.c1_case(order=8)
    else:
        case = synthetic.layered_case(a.config, n_shots=a.shots, nt=a.nt)
    args = (case["grid"], case["geometry"], case["wavelet"], case["config"])
    out = {}
    for res in (-1, 1):
        p = Propagator(*args, dtype="float32", recon="full", resident=res)
        p.set_model(case["true"].m)
        obs = p.synthetic().clone()
        p.set_model(case["init"].m)
        plan = p.resident_plan()
        syn = p.synthetic().clone()
        mis = p.misfit(obs)
        v, g = p.gradient(obs)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.gradient(obs)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        tf = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.misfit(obs)
            e1.record()
            torch.cuda.synchronize()
            tf.append(e0.elapsed_time(e1))
        out[res] = (syn, mis, v, g.clone(), min(ts), min(tf), plan, obs)
        print(f"resident={res}: plan={plan} gradient {min(ts):.2f} ms misfit(fwd) {min(tf):.2f} ms "
              f"value {v:.9e}", flush=True)
    s0, m0, v0, g0, *_ = out[-1]
    s1, m1, v1, g1, *_ = out[1]
    o0, o1 = out[-1][7], out[1][7]
    dg = (g1 - g0).double().norm().item() / max(g0.double().norm().item(), 1e-300)
    print(f"obs bitwise {torch.equal(o0, o1)}  syn bitwise {torch.equal(s0, s1)}  "
          f"misfit equal {m0 == m1}  value rel {abs(v1 - v0) / abs(v0):.3e}  grad rel {dg:.3e}")
    if not torch.equal(s0, s1):
        d = (s1 - s0).abs()
        print("syn max abs diff", d.max().item(), "at", np.unravel_index(int(d.argmax()), d.shape),
              "rel", ((s1 - s0).double().norm() / s0.double().norm()).item())


if __name__ == "__main__":
    main()

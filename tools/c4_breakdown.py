"""Time the pieces of a C4 LSRTM gradient: cached-background and recomputed
(lock-step) shot batches, Born forward vs adjoint.

    python tools/c4_breakdown.py [--nt 6000]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=2):
    import torch
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nt", type=int, default=None)
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case("c4", nt=a.nt)
    args = (case["grid"], case["geometry"], case["wavelet"], case["config"])
    S = case["geometry"].n_sources
    p = Propagator(*args, dtype="float32")
    p.set_model(case["background"].m if "background" in case else case["init"].m)
    m_r = case["reflectivity"].m_r
    d = p.born_forward(m_r).clone()
    print("recon", p.query(), flush=True)
    t_lsrtm_nc = timed(lambda: p.lsrtm_gradient(m_r * 0.5, d))
    t_fwd_nc = timed(lambda: p.born_forward(m_r))
    t_adj_nc = timed(lambda: p.born_adjoint(d))
    print(f"no cache : lsrtm {t_lsrtm_nc:.1f} ms  born_fwd(lockstep) {t_fwd_nc:.1f}  "
          f"born_adj(bg recompute) {t_adj_nc:.1f}", flush=True)
    p.born_cache()
    nc = p.born_cached()
    print("cached shots", nc, flush=True)
    t_lsrtm = timed(lambda: p.lsrtm_gradient(m_r * 0.5, d))
    t_fwd = timed(lambda: p.born_forward(m_r))
    t_adj = timed(lambda: p.born_adjoint(d))
    c0 = nc[0] + nc[1]
    print(f"cache    : lsrtm {t_lsrtm:.1f} ms  born_fwd {t_fwd:.1f}  born_adj {t_adj:.1f}", flush=True)
    for rng in ((0, int(c0)), (int(c0), S)):
        if rng[1] <= rng[0]:
            continue
        shots = (rng[0], rng[1] - rng[0])
        t = timed(lambda: p.lsrtm_gradient(m_r * 0.5, d[rng[0]:rng[1]], shots=shots))
        print(f"  shots {rng}: lsrtm {t:.1f} ms", flush=True)


if __name__ == "__main__":
    main()

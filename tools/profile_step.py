"""Launch the C3 step kernels directly (no graphs) for ncu captures.

    python tools/profile_step.py [--config c3] [--reps 20]

Runs `reps` forward-step (history store) and `reps` adjoint-step (imaging)
launches over all shots of the config, timed with CUDA events."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--recon", default="full")
    ap.add_argument("--shots", type=int, default=None)
    ap.add_argument("--nt", type=int, default=None)
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = (synthetic.layered_case(a.config, n_shots=a.shots, nt=a.nt) if a.config != "c1"
            else synthetic.c1_case())
    prop = Propagator(case["grid"], case["geometry"], case["wavelet"], case["config"],
                      dtype=a.dtype, recon=a.recon, use_graphs=False)
    prop.set_model(case["init"].m)
    S = case["geometry"].n_sources
    bnd = a.recon == "boundary"
    f = prop.time_step_kernel(6 if bnd else 0, S, a.reps)
    b = prop.time_step_kernel(5 if bnd else 1, S, a.reps)
    torch.cuda.synchronize()
    print(f"forward step {f*1e3:.1f} us, adjoint step {b*1e3:.1f} us, shots/launch "
          f"{prop.query()['batch']}")


if __name__ == "__main__":
    main()

"""One FWI gradient of a BASELINE config with plain launches (no CUDA graphs),
for ncu captures inside a real sweep (tools/traffic_capture.sh).

    python tools/one_gradient.py [--config c3] [--shots N] [--nt N] [--recon full]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--shots", type=int, default=None)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--recon", default="auto")
    ap.add_argument("--dtype", default="float32")
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case(a.config, n_shots=a.shots, nt=a.nt)
    prop = Propagator(case["grid"], case["geometry"], case["wavelet"], case["config"],
                      dtype=a.dtype, recon=a.recon, use_graphs=False)
    geom = case["geometry"]
    obs = torch.zeros((geom.n_sources, geom.nt, geom.n_receivers), device="cuda",
                      dtype=prop.tdtype)
    prop.set_model(case["init"].m)
    val, grad = prop.gradient(obs)
    torch.cuda.synchronize()
    print(f"misfit {val:.6e}, recon {prop.query()['recon']}, batch {prop.query()['batch']}")


if __name__ == "__main__":
    main()

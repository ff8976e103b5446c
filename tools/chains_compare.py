"""C3 gradient time with one vs two concurrent half-batch chains.
    python tools/chains_compare.py [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
    case = synthetic.layered_case(cfgname)
    geom = case["geometry"]
    ref = None
    for chains in (1, 2, 3, 4, 2, 3):
        prop = Propagator(case["grid"], geom, case["wavelet"], case["config"], dtype="float32",
                          recon="full", chains=chains)
        prop.set_model(case["true"].m)
        obs = prop.synthetic()
        prop.set_model(case["init"].m)
        v, g = prop.gradient(obs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            v, g = prop.gradient(obs)
        e1.record()
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(3):
            prop.misfit(obs)
        e3.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = g.clone()
        d = float((g - ref).double().norm() / ref.double().norm())
        print(f"chains {chains}: gradient {e0.elapsed_time(e1) / 3:.1f} ms, misfit "
              f"{e2.elapsed_time(e3) / 3:.1f} ms, value {v:.8e}, rel diff {d:.2e}", flush=True)
        del prop
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

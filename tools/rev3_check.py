"""Boundary-saving reversal accuracy at full length: C5 grid (1041x3041
padded), `--shots` shots x nt 12000, fp32.  Prints the relative L2 difference
between the boundary-saving gradient and the checkpointed one (which equals
the stored-history gradient bit for bit), for the library SG_LIB selects
(compare the increment-form and the three-level reversal builds)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shots", type=int, default=2)
    ap.add_argument("--nt", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import synthetic, wavesim
    case = synthetic.layered_case("c5", n_shots=a.shots, nt=a.nt or None)
    args = (case["grid"], case["geometry"], case["wavelet"], case["config"])
    out = {}
    for recon in ("checkpoint", "boundary"):
        p = wavesim.Propagator(*args, dtype="float32", recon=recon)
        p.set_model(case["true"].m)
        obs = p.synthetic()
        p.set_model(case["init"].m)
        v, g = p.gradient(obs)
        out[recon] = (v, g.double().cpu())
        p.close()
        del p
        torch.cuda.empty_cache()
    (v0, g0), (v1, g1) = out["checkpoint"], out["boundary"]
    print(f"C5 grid, {a.shots} shots x nt {case['geometry'].nt}: misfit equal {v0 == v1}, "
          f"boundary vs checkpoint gradient rel L2 {float((g1 - g0).norm() / g0.norm()):.3e}",
          flush=True)


if __name__ == "__main__":
    main()

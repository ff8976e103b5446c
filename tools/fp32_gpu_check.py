"""fp32 production-path accuracy on the GPU against the reference goldens
(run on the GPU box; SG_LIB selects a variant library for A/B):

    python tools/fp32_gpu_check.py

C1 (8th order) fp32 gradient at the reference's AA iterates 0 and 19, the
small 60 x 40 golden, and the fp32 gathers against the fp64 ones.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import torch
    from cases import c1, rel, small_case
    from paper_2008_11778_b200 import gradients
    from paper_2008_11778_b200.wavesim import Propagator
    print("library:", os.environ.get("SG_LIB", "default"))
    case = c1(8)
    g = case["gold"]
    geom, grid = case["geometry"], case["grid"]
    args = (grid, geom, case["wavelet"], case["config"])
    p64 = Propagator(*args, dtype="float64")
    p64.set_model(g["m_true"])
    obs = p64.synthetic().clone()
    keep = list(g["aa_keep"])
    for it in (0, 5, 10, 19):
        if it not in keep:
            continue
        k = keep.index(it)
        obj = gradients.FwiObjective(*args[:1], obs.float(), *args[2:0:-1], case["config"],
                                     dtype="float32")
        val, grad = obj.value_and_grad(g["aa_iterates"][k])
        syn32 = obj.prop.synthetic().double()
        obj.prop.close()
        p64.set_model(g["aa_iterates"][k].reshape(grid.nz, grid.nx))
        syn64 = p64.synthetic()
        de = float(torch.linalg.vector_norm(syn32 - syn64) / torch.linalg.vector_norm(syn64))
        rf = float(torch.linalg.vector_norm(syn64 - obs) / torch.linalg.vector_norm(syn64))
        print(f"C1 iterate {it:2d}: gradient {rel(grad, g['aa_grads'][k]):.2e} misfit "
              f"{abs(val - float(g['aa_values'][k])) / float(g['aa_values'][k]):.2e} "
              f"gathers {de:.2e} residual/data {rf:.2e}")
    p64.close()
    for top in (True, False):
        sc = small_case(8, top)
        gd = sc["gold"]
        pr = Propagator(sc["grid"], sc["geometry"], sc["wavelet"], sc["config"], dtype="float32")
        pr.set_model(sc["model"].m)
        obs_s = torch.as_tensor(np.stack([gd["obs_shot0"], gd["obs_shot1"]])
                                if "obs_shot0" in gd.files else gd["obs"], device="cuda")
        v, gr = pr.gradient(obs_s.float())
        pr.close()
        key = "fwi_grad" if "fwi_grad" in gd.files else "grad"
        print(f"small_o8_{'top' if top else 'free'}: gradient "
              f"{rel(gr.cpu().numpy(), gd[key]):.2e}")


if __name__ == "__main__":
    main()

"""fp32 gradient / Born image error vs the fp64 reference golden on the small
cases and C1, for the current library (SG_LIB selects a variant build):
used to compare the three-level and the V/w increment-form adjoint."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from cases import c1, oracle_setup, rel, small_case  # noqa: E402
from paper_2008_11778_b200 import wavesim  # noqa: E402

for order in (2, 8):
    for top in (True, False):
        case = small_case(order, top)
        g = case["gold"]
        args = (case["grid"], case["geometry"], case["wavelet"], case["config"])
        for mode in (1, 2):
            p = wavesim.Propagator(*args, dtype="float32", recon="full", step_mode=mode)
            p.set_model(g["m"])
            v, gr = p.gradient(g["obs"])
            img = p.born_adjoint(g["y"])
            print(f"small o{order} top={top} step_mode={mode}: grad {rel(gr.cpu().numpy(), g['grad']):.3e} "
                  f"img {rel(img.cpu().numpy(), g['img']):.3e}", flush=True)
case = c1(8)
g = case["gold"]
geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
obs = np.stack(oracle.fwi_synthetic(oracle_setup(g["m_true"], grid, geom, cfg), wav.samples,
                                    geom.nt, threads=5))
p = wavesim.Propagator(grid, geom, wav, cfg, dtype="float32")
p.set_model(g["m_init"])
v, gr = p.gradient(obs)
print(f"C1 fp32 grad {rel(gr.cpu().numpy(), g['grad']):.3e}", flush=True)

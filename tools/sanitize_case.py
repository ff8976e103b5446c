"""Small sweeps for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

The 60 x 40 case of the goldens (2 shots, 28 receivers with a duplicate, 8th
order) cut to `--nt` steps: FWI gradient in FULL / CHECKPOINT / BOUNDARY
reconstruction, fp32 and fp64, two concurrent shot chains, PDL launches (the
library's default launch path), plus the Born/LSRTM gradient (cached and
lock-step backgrounds) and an AA window push/step.  Run on the GPU box as

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

(tools/sanitize.sh runs the four tools and keeps the logs).  Graph capture is
off by default so the sanitizer sees plain launches; --graphs turns it on.
Where compute-sanitizer is not available (this build's GPU pool refuses it),

    SG_REDZONE=1 python tools/sanitize_case.py --redzone [--graphs]

runs the same sweeps on guarded allocations (64 KB of NaN bytes either side of
every device buffer: out-of-bounds reads poison the finite-ness checks below,
out-of-bounds writes are counted by sg_redzone_check).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nt", type=int, default=40)
    ap.add_argument("--graphs", action="store_true")
    ap.add_argument("--dtypes", nargs="+", default=["float32", "float64"])
    ap.add_argument("--recons", nargs="+", default=["full", "checkpoint", "boundary"])
    ap.add_argument("--skip-born", action="store_true")
    ap.add_argument("--skip-aa", action="store_true")
    ap.add_argument("--redzone", action="store_true",
                    help="require SG_REDZONE=1 and check the guard zones at the end "
                         "(the library's own memcheck, include/seisgpu.h)")
    a = ap.parse_args()
    import torch
    from paper_2008_11778_b200 import anderson
    from paper_2008_11778_b200.model import AcquisitionGeometry, Grid2D, SimConfig, make_ricker
    from paper_2008_11778_b200.wavesim import Propagator
    from cases import small_geometry

    g0 = small_geometry()
    geom = AcquisitionGeometry(g0.sources, g0.receivers, dt=g0.dt, nt=a.nt)
    grid = Grid2D(nx=60, nz=40, dx=20.0, dz=20.0)
    wav = make_ricker(12.0, geom.dt, a.nt, t0=0.02)
    cfg = SimConfig(border_width=10, damp_top=True, order=8)
    rng = np.random.default_rng(0)
    z = np.linspace(0.0, 1.0, grid.nz)[:, None]
    m = (1.0 / (1800.0 + 900.0 * z + 40.0 * rng.standard_normal((grid.nz, grid.nx)))) ** 2
    m_true = (1.0 / (1800.0 + 1100.0 * z + 0.0 * m)) ** 2
    m_r = 1e-8 * rng.standard_normal((grid.nz, grid.nx))
    for dtype in a.dtypes:
        for recon in a.recons:
            prop = Propagator(grid, geom, wav, cfg, dtype=dtype, recon=recon, chains=2,
                              use_graphs=a.graphs, checkpoint_every=7 if recon == "checkpoint" else 0)
            prop.set_model(m_true)
            obs = prop.synthetic()
            prop.set_model(m)
            val = prop.misfit(obs)
            val2, grad = prop.gradient(obs)
            torch.cuda.synchronize()
            assert np.isfinite(val) and abs(val - val2) <= 1e-5 * abs(val), (val, val2)
            assert bool(torch.isfinite(grad).all())
            if not a.skip_born and recon != "boundary":
                d_r = prop.born_forward(m_r)              # lock-step background
                v1, g1 = prop.lsrtm_gradient(np.zeros_like(m_r), d_r)
                prop.born_cache()                          # cached background histories
                d_c = prop.born_forward(m_r)
                v2, g2 = prop.lsrtm_gradient(np.zeros_like(m_r), d_c)
                torch.cuda.synchronize()
                assert np.isfinite(v1) and np.isfinite(v2)
                assert bool(torch.isfinite(g1).all()) and bool(torch.isfinite(g2).all())
            print(f"{dtype} {recon}: misfit {val:.6e} |grad| {float(grad.norm()):.6e}", flush=True)
            prop.close()
    if not a.skip_aa:
        n, mm = 6000, 5
        for dtype in a.dtypes:
            win = anderson.AAWindow(n, mm, dtype=dtype)
            out = torch.empty(n, device="cuda", dtype=win.tdtype if hasattr(win, "tdtype")
                              else getattr(torch, dtype))
            tg = torch.Generator(device="cuda")
            tg.manual_seed(1)
            for _ in range(mm + 3):
                p = torch.randn(n, generator=tg, device="cuda", dtype=out.dtype)
                gq = p * 0.5 + 0.1 * torch.randn(n, generator=tg, device="cuda", dtype=out.dtype)
                win.push(p, gq)
                if win.m_k:
                    anderson.aa_step(win, weights=anderson.aa_weights(win), out=out)
            torch.cuda.synchronize()
            assert bool(torch.isfinite(out).all())
            print(f"AA window {dtype}: ok", flush=True)
    if a.redzone:
        from paper_2008_11778_b200 import _lib
        import gc
        gc.collect()
        bad, n = _lib.redzone_check()
        assert n > 0, "SG_REDZONE=1 was not set when the library was loaded"
        assert bad == 0, f"{bad} guard bytes modified: out-of-bounds write"
        # self-test: a byte written past a live allocation must be found
        keep = anderson.AAWindow(1000, 2, dtype="float32")
        bad2, n2 = _lib.redzone_check(poke=True)
        assert bad2 == 1 and n2 > n, (bad2, n2)
        del keep
        print(f"redzone: {n} guarded allocations, 0 guard bytes modified; self-test poke found")
    print("sanitize_case: done")


if __name__ == "__main__":
    main()

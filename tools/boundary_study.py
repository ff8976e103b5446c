"""Accuracy study of boundary-saving reconstruction (NumPy emulation, CPU).

The forward keeps only the final state (u_nt, inc_nt) and, per step, u_n on
the sponge band (cells with damp < 1).  The adjoint then runs the forward
backwards in the undamped interior,
    a_n = inv_m L u_n (+ source),  inc_n = inc_{n+1} - dt^2 a_n,
    u_{n-1} = u_n - inc_n,
takes band cells from the store, and images against the reconstructed a_n.
Reports the gradient error of (stored history) and (reconstructed) against
the fp64 reference golden, in fp32 and fp64.
Usage: python tools/boundary_study.py [c1|c3]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tools")]
import oracle  # noqa: E402
from cases import c1, oracle_setup  # noqa: E402
from fp32_study import lap  # noqa: E402


def run(st, obs, wav, nt, dtype, recon, shots=None):
    c8 = oracle.LAP8
    cz = [dtype(c * st.kz) for c in c8]
    cx = [dtype(c * st.kx) for c in c8]
    im = st.inv_m.astype(dtype)
    d = st.damp.astype(dtype)
    band = st.damp < 1.0
    dt2 = dtype(st.dt2)
    coef = dt2 * im * d
    rr, rc, rw = st.rec
    rw = rw.astype(dtype)
    wq = oracle.trapezoid(nt)
    grad = np.zeros(st.shape, dtype)
    val = 0.0
    worst = 0.0
    for s in (range(st.n_sources) if shots is None else shots):
        sr, sc = st.src[0][:, s], st.src[1][:, s]
        sw = (st.src[2][:, s] * st.src_scale).astype(dtype)

        def accel(u, n):
            a = lap(u, cz, cx, "diff") * im
            for t in range(4):
                a[sr[t], sc[t]] += dtype(wav[n]) * sw[t] * im[sr[t], sc[t]]
            return a

        u = np.zeros(st.shape, dtype)
        inc = np.zeros(st.shape, dtype)
        hist = None if recon else np.empty((nt, *st.shape), dtype)
        bstore = np.empty((nt, int(band.sum())), dtype) if recon else None
        tr = np.zeros((nt, st.n_receivers), dtype)
        ref_a = []
        for n in range(nt):
            tr[n] = (rw * u[rr, rc]).sum(axis=0)
            a = accel(u, n)
            if recon:
                bstore[n] = u[band]
                if n % 500 == 0:
                    ref_a.append((n, a.copy()))
            else:
                hist[n] = a
            inc = d * (inc + dt2 * a)
            u = d * u + inc
        res = tr - obs[s].astype(dtype)
        val += 0.5 * st.dt * float(np.sum(wq[:, None] * res.astype(np.float64) ** 2))
        yb = (wq[:, None] * st.dt).astype(dtype) * res
        V = np.zeros(st.shape, dtype)
        w = np.zeros(st.shape, dtype)
        img = np.zeros(st.shape, dtype)
        if recon:
            # state (u_n, inc_{n+1}) for n = nt-1: u_{nt-1} = u_nt - inc_nt inside
            un = u - inc
            un[band] = bstore[nt - 1]
            incn1 = inc
        checks = dict(ref_a)
        for n in range(nt - 1, -1, -1):
            if recon:
                a = accel(un, n)
                if n in checks:
                    e = np.linalg.norm(a - checks[n]) / max(np.linalg.norm(checks[n]), 1e-300)
                    worst = max(worst, e)
                incn = incn1 - dt2 * a
                if n > 0:
                    un = un - incn
                    un[band] = bstore[n - 1]
                incn1 = incn
            else:
                a = hist[n]
            L = lap(V, cz, cx, "diff")
            inj = np.zeros(st.shape, dtype)
            np.add.at(inj, (rr, rc), rw * yb[n])
            w = d * w + (L + inj)
            img -= a * V
            V = d * V + coef * w
        grad += img
    return val, oracle.fold_pad(grad.astype(np.float64), st.pads, st.nz, st.nx), worst


def main():
    case = c1(8)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st_true = oracle_setup(g["m_true"], grid, geom, cfg)
    obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt, threads=5)
    st = oracle_setup(g["m_init"], grid, geom, cfg)
    for dtype in (np.float32, np.float64):
        for recon in (False, True):
            v, gr, worst = run(st, obs, wav.samples, geom.nt, dtype, recon)
            e = np.linalg.norm(gr - g["grad"]) / np.linalg.norm(g["grad"])
            print(f"{dtype.__name__} recon={recon}: misfit err {abs(v - g['value']) / g['value']:.2e}"
                  f"  grad err {e:.2e}  worst accel err {worst:.2e}", flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def c3_one_shot():
    """One C3 shot (nt 4000): fp32 recon and fp32 stored vs fp64 stored."""
    from paper_2008_11778_b200 import synthetic
    case = synthetic.layered_case("c3", n_shots=30)
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st_true = oracle_setup(case["true"].m, grid, geom, cfg)
    obs = [None] * 30
    obs[15] = oracle.forward_sweep(st_true, geom.nt, wav.samples, shot=15, keep=False)[0]
    st = oracle_setup(case["init"].m, grid, geom, cfg)
    v64, g64, _ = run(st, obs, wav.samples, geom.nt, np.float64, False, shots=[15])
    for recon in (False, True):
        v, gr, worst = run(st, obs, wav.samples, geom.nt, np.float32, recon, shots=[15])
        e = np.linalg.norm(gr - g64) / np.linalg.norm(g64)
        print(f"C3 shot 15 fp32 recon={recon}: misfit err {abs(v - v64) / v64:.2e} grad err {e:.2e}"
              f" worst accel err {worst:.2e}", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c3":
    c3_one_shot()

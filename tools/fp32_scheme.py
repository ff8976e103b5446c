"""fp32 forward schemes for the production path (NumPy emulation, CPU).

tools/fp32_budget.py shows that the fp32 gradient error lives in the forward
sweep, and single-rounding-point experiments at C1 AA iterate 19 (where the
residual is ~1.5e-3 of the data) rank the sources: the fp32 rounding of the
global stencil weights c_k / h^2 (a coherent velocity bias, 8e-4), then the
storage rounding of u and inc (1e-4 each), of 1/m per cell (8e-5) and of dt^2
(4e-5); the fp32 Laplacian arithmetic itself is benign (3e-5).

Schemes emulated here (every operation rounded to fp32 as the device does;
fma = one rounding):
  base   the round-1 kernel: a = (sum_k cz_k dz_k + cx_k dx_k) * (1/m);
         inc' = d (inc + dt2 a); u' = d u + inc'
  ratio  weights as exact ratios r_k = c_k / c_1 (r_2 = -1/8 exact) and
         per-cell w = c_1 kz / m split hi + lo (two fp32 planes), dt2 split
         hi + lo: a = lp w_hi + lp w_lo, dta = dt2_hi a + dt2_lo a
  +carry the same with compensated (two-sum) updates of inc and u; the carries
         are stored per cell (fp32, or bf16 with 'h')

    python tools/fp32_scheme.py [--iterates 0 19] [--schemes base ratio ratio+carry ...]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tools")]
import oracle  # noqa: E402
from cases import c1, oracle_setup  # noqa: E402
from fp32_budget import adjoint, bf16  # noqa: E402
from fp32_study import shift  # noqa: E402

F = np.float32
D = np.float64


def fma(a, b, c):
    return (np.asarray(a, D) * np.asarray(b, D) + np.asarray(c, D)).astype(F)


def split(x):
    hi = np.asarray(x, D).astype(F)
    lo = (np.asarray(x, D) - hi.astype(D)).astype(F)
    return hi, lo


def forward(st, wav, nt, s, scheme):
    c8 = oracle.LAP8
    d = st.damp.astype(F)
    rr, rc, rw = st.rec
    rw = rw.astype(F)
    sr, sc = st.src[0][:, s], st.src[1][:, s]
    swd = st.src[2][:, s] * st.src_scale
    carry = "carry" in scheme
    q16 = bf16 if scheme.endswith("h") else (lambda x: x)
    u = np.zeros(st.shape, F)
    inc = np.zeros(st.shape, F)
    ul = np.zeros(st.shape, F)
    il = np.zeros(st.shape, F)
    hist = np.empty((nt, *st.shape), F)
    tr = np.zeros((nt, st.n_receivers), F)
    if scheme == "base":
        cz = [F(c * st.kz) for c in c8]
        cx = [F(c * st.kx) for c in c8]
        im = st.inv_m.astype(F)
        dt2 = F(st.dt2)
    else:
        c1 = c8[1]
        r = [F(c / c1) for c in c8]            # r_1 = 1, r_2 = -1/8 exact
        rho = F(st.kx / st.kz)                 # 1 when dx == dz
        w_hi, w_lo = split(c1 * st.kz * st.inv_m)
        dt2_hi, dt2_lo = split(st.dt2)
        swp = swd / (c1 * st.kz)               # source weight on the w scale
    for n in range(nt):
        tr[n] = (rw * u[rr, rc]).sum(axis=0)
        if scheme == "base":
            lz = np.zeros(st.shape, F)
            lx = np.zeros(st.shape, F)
            for k in range(1, 5):
                lz = fma(cz[k], (shift(u, k, 0) - u) + (shift(u, -k, 0) - u), lz)
                lx = fma(cx[k], (shift(u, k, 1) - u) + (shift(u, -k, 1) - u), lx)
            a = (lz + lx) * im
            for t in range(4):
                a[sr[t], sc[t]] += F(wav[n]) * F(swd[t]) * im[sr[t], sc[t]]
            dta = dt2 * a
        else:
            lz = np.zeros(st.shape, F)
            lx = np.zeros(st.shape, F)
            for k in range(1, 5):
                lz = fma(r[k], (shift(u, k, 0) - u) + (shift(u, -k, 0) - u), lz)
                lx = fma(r[k], (shift(u, k, 1) - u) + (shift(u, -k, 1) - u), lx)
            lp = fma(rho, lx, lz)
            a = fma(lp, w_hi, lp * w_lo)
            for t in range(4):
                a[sr[t], sc[t]] += F(wav[n]) * F(swp[t]) * w_hi[sr[t], sc[t]]
            dta = fma(dt2_hi, a, dt2_lo * a)
        hist[n] = a
        if carry:
            # inc' = d (inc + il + dta) as a two-sum (carry il), then u' = d u + inc'
            y = dta + il
            t = inc + y
            il = q16(y - (t - inc))
            inc = d * t
            il = q16(d * il)
            du = d * u
            y = inc + il + ul
            t = du + y
            ul = q16(y - (t - du))
            u = t
        else:
            inc = d * (inc + dta)
            u = d * u + inc
    return tr, hist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterates", type=int, nargs="+", default=[0, 19])
    ap.add_argument("--schemes", nargs="+", default=["base", "ratio", "ratio+carry",
                                                      "ratio+carryh"])
    a = ap.parse_args()
    case = c1(8)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    obs = oracle.fwi_synthetic(oracle_setup(g["m_true"], grid, geom, cfg), wav.samples,
                               geom.nt, threads=5)
    keep = list(g["aa_keep"])
    wq = oracle.trapezoid(geom.nt)
    for it in a.iterates:
        st = oracle_setup(g["aa_iterates"][keep.index(it)].reshape(grid.nz, grid.nx), grid,
                          geom, cfg)
        ref_v, ref_g = oracle.fwi_gradient(st, obs, wav.samples, geom.nt, threads=5)[:2]
        for sch in a.schemes:
            grad = np.zeros(st.shape)
            val = 0.0
            for s in range(geom.n_sources):
                tr, hist = forward(st, wav.samples, geom.nt, s, sch)
                res = (tr - obs[s].astype(F)).astype(D)
                val += 0.5 * st.dt * float(np.sum(wq[:, None] * res ** 2))
                grad += adjoint(st, (wq[:, None] * st.dt) * res, hist, F).astype(D)
            gr = oracle.fold_pad(grad, st.pads, st.nz, st.nx)
            e = np.linalg.norm(gr - ref_g) / np.linalg.norm(ref_g)
            print(f"iterate {it:2d} {sch:14s} misfit {abs(val - ref_v) / ref_v:.2e} "
                  f"grad {e:.2e}", flush=True)


if __name__ == "__main__":
    main()

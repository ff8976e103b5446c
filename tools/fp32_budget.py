"""Where the fp32 gradient error comes from (NumPy emulation of the device
recursion, CPU) -- and what a compensated forward buys.

For C1 (8th order) at the reference's AA iterates 0 and 19 (c1_o8.npz), the
gradient is computed with the forward and the adjoint each in fp32 or fp64:

  fwd32/adj32  the device's fp32 production path
  fwd64/adj32  exact forward (gathers, history) + fp32 adjoint
  fwd32/adj64  fp32 forward + exact adjoint
  kahan/adj32  fp32 forward with a compensated field update
               (u_{n+1} = u_n + inc_{n+1} summed with a Kahan carry c per cell,
               c stored as fp32 / bf16) + fp32 adjoint

    python tools/fp32_budget.py [--iterates 0 19] [--shots 5]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
from cases import c1, oracle_setup  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tools"))
from fp32_study import lap  # noqa: E402


def bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def forward(st, wav, nt, s, dt, mode):
    """Gathers and acceleration history of shot s.  mode: 'f32', 'f64',
    'kahan32' (fp32 carry), 'kahan16' (bf16 carry)."""
    c8 = oracle.LAP8
    cz = [dt(c * st.kz) for c in c8]
    cx = [dt(c * st.kx) for c in c8]
    im = st.inv_m.astype(dt)
    d = st.damp.astype(dt)
    dt2 = dt(st.dt2)
    rr, rc, rw = st.rec
    rw = rw.astype(dt)
    sr, sc, sw = st.src[0][:, s], st.src[1][:, s], (st.src[2][:, s] * st.src_scale).astype(dt)
    u = np.zeros(st.shape, dt)
    inc = np.zeros(st.shape, dt)
    c = np.zeros(st.shape, dt)
    hist = np.empty((nt, *st.shape), dt)
    tr = np.zeros((nt, st.n_receivers), dt)
    for n in range(nt):
        tr[n] = (rw * u[rr, rc]).sum(axis=0)
        a = lap(u, cz, cx, "diff") * im
        for t in range(4):
            a[sr[t], sc[t]] += dt(wav[n]) * sw[t] * im[sr[t], sc[t]]
        hist[n] = a
        inc = d * (inc + dt2 * a)
        if mode.startswith("kahan"):
            # u' = d u + inc' with a running carry: y = inc' - c,
            # t = du + y, c = (t - du) - y
            du = d * u
            y = inc - c
            t = du + y
            c = (t - du) - y
            if mode == "kahan16":
                c = bf16(c)
            u = t
        else:
            u = d * u + inc
    return tr, hist


def adjoint(st, yb, hist, dt):
    c8 = oracle.LAP8
    cz = [dt(c * st.kz) for c in c8]
    cx = [dt(c * st.kx) for c in c8]
    im = st.inv_m.astype(dt)
    d = st.damp.astype(dt)
    dt2 = dt(st.dt2)
    coef = dt2 * im * d
    rr, rc, rw = st.rec
    rw = rw.astype(dt)
    nt = yb.shape[0]
    yb = yb.astype(dt)
    hist = hist.astype(dt)
    V = np.zeros(st.shape, dt)
    Vp = np.zeros(st.shape, dt)
    img = np.zeros(st.shape, dt)
    for n in range(nt - 1, -1, -1):
        L = lap(V, cz, cx, "diff")
        inj = np.zeros(st.shape, dt)
        np.add.at(inj, (rr, rc), rw * yb[n])
        img -= hist[n] * V
        Vn = coef * (L + inj) + d * ((V + V) - d * Vp)  # three-level (device default)
        Vp, V = V, Vn
    return img


def gradient(st, obs, wav, nt, fwd_mode, adj_dt, shots):
    wq = oracle.trapezoid(nt)
    grad = np.zeros(st.shape)
    val = 0.0
    fdt = np.float64 if fwd_mode == "f64" else np.float32
    for s in shots:
        tr, hist = forward(st, wav, nt, s, fdt, fwd_mode)
        res = tr.astype(np.float64) - obs[s]
        if fdt == np.float32:
            res = (tr - obs[s].astype(np.float32)).astype(np.float64)
        val += 0.5 * st.dt * float(np.sum(wq[:, None] * res ** 2))
        yb = (wq[:, None] * st.dt) * res
        grad += adjoint(st, yb, hist, adj_dt).astype(np.float64)
    return val, oracle.fold_pad(grad, st.pads, st.nz, st.nx)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterates", type=int, nargs="+", default=[0, 19])
    ap.add_argument("--shots", type=int, default=5)
    ap.add_argument("--modes", nargs="+",
                    default=["f32/32", "f64/32", "f32/64", "kahan32/32", "kahan16/32"])
    a = ap.parse_args()
    case = c1(8)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st_true = oracle_setup(g["m_true"], grid, geom, cfg)
    obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt, threads=5)
    keep = list(g["aa_keep"])
    shots = list(range(a.shots))
    for it in a.iterates:
        k = keep.index(it)
        m = g["aa_iterates"][k].reshape(grid.nz, grid.nx)
        st = oracle_setup(m, grid, geom, cfg)
        ref_v, ref_g = oracle.fwi_gradient(st, obs, wav.samples, geom.nt, threads=5,
                                           shots=shots)[:2]
        for mode in a.modes:
            fm, am = mode.split("/")
            v, gr = gradient(st, obs, wav.samples, geom.nt, fm,
                             np.float64 if am == "64" else np.float32, shots)
            e = np.linalg.norm(gr - ref_g) / np.linalg.norm(ref_g)
            print(f"iterate {it:2d} fwd {fm:8s} adj {am}: misfit {abs(v - ref_v) / ref_v:.2e} "
                  f"grad {e:.2e}", flush=True)


if __name__ == "__main__":
    main()

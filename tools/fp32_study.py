"""fp32 accuracy study of the GPU recursion (NumPy emulation, CPU).

Emulates the device algorithm (increment-form leapfrog, V-form adjoint,
imaging) in float32 with two Laplacian evaluation orders and reports the
gradient error against the fp64 reference golden for C1 (8th order):
  diff : sum_k c_k ((u_{+k}-u) + (u_{-k}-u))      (current kernel)
  std  : c_0 u + sum_k c_k (u_{+k} + u_{-k})
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
from cases import c1, oracle_setup  # noqa: E402

F = np.float32


def shift(u, k, axis):
    out = np.zeros_like(u)
    if axis == 0:
        if k > 0:
            out[:-k] = u[k:]
        else:
            out[-k:] = u[:k]
    else:
        if k > 0:
            out[:, :-k] = u[:, k:]
        else:
            out[:, -k:] = u[:, :k]
    return out


def lap(u, cz, cx, form):
    if form == "diff":
        lz = np.zeros_like(u)
        lx = np.zeros_like(u)
        for k in range(1, 5):
            lz += cz[k] * ((shift(u, k, 0) - u) + (shift(u, -k, 0) - u))
            lx += cx[k] * ((shift(u, k, 1) - u) + (shift(u, -k, 1) - u))
        return lz + lx
    out = (cz[0] + cx[0]) * u
    for k in range(1, 5):
        out = out + cz[k] * (shift(u, k, 0) + shift(u, -k, 0))
        out = out + cx[k] * (shift(u, k, 1) + shift(u, -k, 1))
    return out


def run(st, obs, wav, nt, form, dtype=F):
    c8 = oracle.LAP8
    cz = [dtype(c * st.kz) for c in c8]
    cx = [dtype(c * st.kx) for c in c8]
    im = st.inv_m.astype(dtype)
    d = st.damp.astype(dtype)
    dt2 = dtype(st.dt2)
    coef = dt2 * im * d
    rr, rc, rw = st.rec
    rw = rw.astype(dtype)
    wq = oracle.trapezoid(nt)
    grad = np.zeros(st.shape, dtype)
    val = 0.0
    for s in range(st.n_sources):
        sr, sc, sw = st.src[0][:, s], st.src[1][:, s], (st.src[2][:, s] * st.src_scale).astype(dtype)
        u = np.zeros(st.shape, dtype)
        inc = np.zeros(st.shape, dtype)
        hist = np.empty((nt, *st.shape), dtype)
        tr = np.zeros((nt, st.n_receivers), dtype)
        for n in range(nt):
            tr[n] = (rw * u[rr, rc]).sum(axis=0)
            a = lap(u, cz, cx, form) * im
            for t in range(4):
                a[sr[t], sc[t]] += dtype(wav[n]) * sw[t] * im[sr[t], sc[t]]
            hist[n] = a
            inc = d * (inc + dt2 * a)
            u = d * u + inc
        res = tr - obs[s].astype(dtype)
        val += 0.5 * st.dt * float(np.sum(wq[:, None] * res.astype(np.float64) ** 2))
        yb = (wq[:, None] * st.dt).astype(dtype) * res
        V = np.zeros(st.shape, dtype)
        w = np.zeros(st.shape, dtype)
        img = np.zeros(st.shape, dtype)
        for n in range(nt - 1, -1, -1):
            L = lap(V, cz, cx, form)
            inj = np.zeros(st.shape, dtype)
            np.add.at(inj, (rr, rc), rw * yb[n])
            w = d * w + (L + inj)
            img -= hist[n] * V
            V = d * V + coef * w
        grad += img
    return val, oracle.fold_pad(grad.astype(np.float64), st.pads, st.nz, st.nx)


def main():
    case = c1(8)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st_true = oracle_setup(g["m_true"], grid, geom, cfg)
    obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt, threads=5)
    st = oracle_setup(g["m_init"], grid, geom, cfg)
    for form in ("diff", "std"):
        v, gr = run(st, obs, wav.samples, geom.nt, form)
        e = np.linalg.norm(gr - g["grad"]) / np.linalg.norm(g["grad"])
        print(f"{form}: misfit rel err {abs(v - g['value']) / g['value']:.2e}  grad rel err {e:.2e}",
              flush=True)
    v, gr = run(st, obs, wav.samples, geom.nt, "diff", dtype=np.float64)
    e = np.linalg.norm(gr - g["grad"]) / np.linalg.norm(g["grad"])
    print(f"fp64 emulation (algorithm check): grad rel err {e:.2e}")


if __name__ == "__main__":
    main()

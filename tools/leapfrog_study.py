"""fp32 study (NumPy emulation, CPU) of three-level leapfrog forms on C1
(8th order): gradient error vs the fp64 golden with the increment-form
forward ("inc") or the reference-order three-level forward ("lf3"), both with
the three-level adjoint.  Result (r01e): inc 3.18e-5, lf3 6.65e-5 (the
three-level adjoint alone leaves the error unchanged: 3.19e-5 with the V/w
form)."""
import sys; sys.path[:0]=['/root/repo/tools','/root/repo','/root/repo/tests']
import numpy as np, fp32_study as fs, oracle
from cases import c1, oracle_setup
F=np.float32
def run(st, obs, wav, nt, scheme, adj3=False):
    c8 = oracle.LAP8; dtype=F
    cz = [dtype(c * st.kz) for c in c8]; cx = [dtype(c * st.kx) for c in c8]
    im = st.inv_m.astype(dtype); d = st.damp.astype(dtype); dt2 = dtype(st.dt2)
    coef = dt2 * im * d
    rr, rc, rw = st.rec; rw = rw.astype(dtype)
    wq = oracle.trapezoid(nt); grad = np.zeros(st.shape, dtype); val = 0.0
    for s in range(st.n_sources):
        sr, sc, sw = st.src[0][:, s], st.src[1][:, s], (st.src[2][:, s] * st.src_scale).astype(dtype)
        u = np.zeros(st.shape, dtype); inc = np.zeros(st.shape, dtype); um1 = np.zeros(st.shape, dtype)
        hist = np.empty((nt, *st.shape), dtype); tr = np.zeros((nt, st.n_receivers), dtype)
        for n in range(nt):
            tr[n] = (rw * u[rr, rc]).sum(axis=0)
            a = fs.lap(u, cz, cx, "diff") * im
            for t in range(4):
                a[sr[t], sc[t]] += dtype(wav[n]) * sw[t] * im[sr[t], sc[t]]
            hist[n] = a
            if scheme == "inc":
                inc = d * (inc + dt2 * a); u = d * u + inc
            elif scheme == "lf3":   # reference order: d*(2u - d*u_{n-1} + dt2*a)
                un = d * (dtype(2) * u - d * um1 + dt2 * a); um1 = u; u = un
            else:  # lf3b: d*((u - d*u_{n-1}) + (u + dt2*a))
                un = d * ((u - d * um1) + dt2 * a + u); um1 = u; u = un
        res = tr - obs[s].astype(dtype)
        val += 0.5 * st.dt * float(np.sum(wq[:, None] * res.astype(np.float64) ** 2))
        yb = (wq[:, None] * st.dt).astype(dtype) * res
        V = np.zeros(st.shape, dtype); w = np.zeros(st.shape, dtype); img = np.zeros(st.shape, dtype); Vp = np.zeros(st.shape, dtype)
        for n in range(nt - 1, -1, -1):
            L = fs.lap(V, cz, cx, "diff"); inj = np.zeros(st.shape, dtype)
            np.add.at(inj, (rr, rc), rw * yb[n])
            if adj3:
                img -= hist[n] * V
                Vm = coef * (L + inj) + (F(2) * d) * V - (d * d) * Vp
                Vp = V; V = Vm
            else:
                w = d * w + (L + inj); img -= hist[n] * V; V = d * V + coef * w
        grad += img
    return val, oracle.fold_pad(grad.astype(np.float64), st.pads, st.nz, st.nx)
case = c1(8); g = case["gold"]
geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
obs = oracle.fwi_synthetic(oracle_setup(g["m_true"], grid, geom, cfg), wav.samples, geom.nt, threads=5)
st = oracle_setup(g["m_init"], grid, geom, cfg)
for sch, a3 in (("inc", True), ("lf3", True)):
    v, gr = run(st, obs, wav.samples, geom.nt, sch, a3)
    print(sch, a3, abs(v-g["value"])/g["value"], np.linalg.norm(gr-g["grad"])/np.linalg.norm(g["grad"]), flush=True)

"""fp32 study (NumPy emulation, CPU) of boundary-saving reversal at C3 (one
shot, 4000 steps): gradient error vs the fp64 oracle with the stored history,
with the increment-form reversal the fused kernel runs
(u_{n-1} = u_n - inc_n, inc_{n-1} = inc_n - dt^2 a_{n-1}), and with a
three-level reversal (u_{n-1} = 2u_n + dt^2 a_n - u_{n+1}); frame cells from
the band store in both.  Result (r01e): 1.34e-6 / 1.42e-6 / 5.58e-6."""
import sys; sys.path[:0]=['/root/repo/tools','/root/repo','/root/repo/tests']
import numpy as np, oracle, time
import fp32_study as fs
from cases import oracle_setup
from paper_2008_11778_b200 import synthetic
from paper_2008_11778_b200.model import AcquisitionGeometry
F=np.float32
case = synthetic.layered_case("c3"); g0 = case["geometry"]
geom = AcquisitionGeometry((g0.sources[11],), g0.receivers, g0.dt, g0.nt)
grid, cfg, wav = case["grid"], case["config"], case["wavelet"]
obs = oracle.fwi_synthetic(oracle_setup(case["true"].m, grid, geom, cfg), wav.samples, geom.nt)
st = oracle_setup(case["init"].m, grid, geom, cfg)
val, grad, _ = oracle.fwi_gradient(st, obs, wav.samples, geom.nt)
nt = geom.nt; w = wav.samples
c8 = oracle.LAP8
cz = [F(c * st.kz) for c in c8]; cx = [F(c * st.kx) for c in c8]
im = st.inv_m.astype(F); d = st.damp.astype(F); dt2 = F(st.dt2); coef = dt2 * im * d
band = d < 1
rr, rc, rw = st.rec; rw = rw.astype(F)
sr, sc, sw = st.src[0][:, 0], st.src[1][:, 0], (st.src[2][:, 0] * st.src_scale).astype(F)
def accel(u, n):
    a = fs.lap(u, cz, cx, "diff") * im
    for t in range(4):
        a[sr[t], sc[t]] += F(w[n]) * sw[t] * im[sr[t], sc[t]]
    return a
u = np.zeros(st.shape, F); inc = np.zeros(st.shape, F)
store = np.empty((nt, int(band.sum())), F); tr = np.zeros((nt, st.n_receivers), F)
hist = np.empty((nt, *st.shape), F)
for n in range(nt):
    tr[n] = (rw * u[rr, rc]).sum(axis=0)
    store[n] = u[band]
    a = accel(u, n); hist[n] = a
    inc = d * (inc + dt2 * a); u = d * u + inc
wq = oracle.trapezoid(nt)
res = tr - obs[0].astype(F)
yb = (wq[:, None] * st.dt).astype(F) * res
def adjoint(get_a):
    V = np.zeros(st.shape, F); Wt = np.zeros(st.shape, F); img = np.zeros(st.shape, F)
    for n in range(nt - 1, -1, -1):
        a_n = get_a(n)
        L = fs.lap(V, cz, cx, "diff"); inj = np.zeros(st.shape, F)
        np.add.at(inj, (rr, rc), rw * yb[n])
        Wt = d * Wt + (L + inj); img -= a_n * V; V = d * V + coef * Wt
    return oracle.fold_pad(img.astype(np.float64), st.pads, st.nz, st.nx)
e = lambda g: np.linalg.norm(g - grad) / np.linalg.norm(grad)
print("stored history", e(adjoint(lambda n: hist[n])), flush=True)
# inc-form reversal: state (u_n, inc_{n+1}) walking down; starts from final u_nt, inc_nt
class IncRev:
    def __init__(s): s.u = u.copy(); s.inc = inc.copy(); s.n = nt
    def __call__(s, n):
        # bring s.u to u_n: u_{m-1} = u_m - inc_m, frame from store
        while s.n > n:
            um = s.u - s.inc
            um[band] = store[s.n - 1]
            # inc_{m-1} = inc_m / d - dt2 a_{m-1} : interior (d=1): inc_m - dt2 a_{m-1}
            a = accel(um, s.n - 1)
            s.inc = s.inc - dt2 * a
            s.u = um; s.n -= 1; s.a = a
        return s.a
print("inc reversal", e(adjoint(IncRev())), flush=True)
class Rev3:
    def __init__(s):
        s.up = u.copy()          # u_nt
        um = u - inc; um[band] = store[nt - 1]
        s.u = um; s.n = nt - 1; s.a = accel(um, nt - 1)   # u_{nt-1}, a_{nt-1}
    def __call__(s, n):
        while s.n > n:
            um = F(2) * s.u + dt2 * s.a - s.up
            um[band] = store[s.n - 1]
            s.up = s.u; s.u = um; s.n -= 1; s.a = accel(um, s.n)
        return s.a
print("3-level reversal", e(adjoint(Rev3())), flush=True)

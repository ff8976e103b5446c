"""NumPy restatement of the seisopt hot path -- the CPU oracle.

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
(as the checker) and ``bench.py`` (``cpu_baseline`` / ``--impl reference``).
The shipped package never imports it and never falls back to it.

Every routine restates the algorithm of the reference package ``seisopt``
(``/root/reference/pkg/src/seisopt``, abbreviated ``seisopt/`` below) with the
same floating-point operation order, so that in fp64 with the 2nd-order stencil
it reproduces the reference bit for bit (pinned by ``tests/golden``).

Deliberate extension: ``order=8`` swaps the 5-point
Laplacian of ``seisopt/wavesim.py:216-223`` for the symmetric 8th-order
zero-exterior Laplacian used by the BASELINE configs, and tightens the CFL bound
of ``seisopt/wavesim.py:92-100`` by sqrt(4 / 6.5016).  The goldens for that
variant are produced by running the reference with the same one-method
substitution (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.linalg import solve_triangular

# 8th-order central second-derivative weights (unit spacing), k = 0..4.
LAP8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)
# Nyquist symbol |sum_k c_k (-1)^k| * ... of the 8th-order operator, per axis.
LAP8_SYMBOL = -(LAP8[0] + 2.0 * sum(c * (-1.0) ** k for k, c in enumerate(LAP8) if k))
CFL8_FACTOR = math.sqrt(4.0 / LAP8_SYMBOL)  # 0.7844: 8th-order / 2nd-order bound


class OracleStabilityError(Exception):
    """CFL violation (mirrors seisopt/wavesim.py:41-42)."""


class OracleEmptyWindow(Exception):
    """Empty AA window (mirrors seisopt/optim/qr.py:18-19)."""


# ---------------------------------------------------------------------------
# Grid set-up: pads, sponge, bilinear taps (seisopt/wavesim.py:108-214)
# ---------------------------------------------------------------------------


def pad_widths(border: int, damp_top: bool = True):
    """(top, bottom, left, right) -- seisopt/wavesim.py:121-123."""
    return (border if damp_top else 0, border, border, border)


def extend_to_pad(values, pads):
    """Edge replication onto the padded grid -- seisopt/wavesim.py:126-128."""
    t, b, l, r = pads
    return np.pad(values, ((t, b), (l, r)), mode="edge")


def fold_pad(padded, pads, nz, nx):
    """Transpose of extend_to_pad -- seisopt/wavesim.py:135-147."""
    t, b, l, r = pads
    g = np.array(padded, copy=True)
    if t:
        g[t] += g[:t].sum(axis=0)
    if b:
        g[-b - 1] += g[-b:].sum(axis=0)
    g = g[t : t + nz]
    if l:
        g[:, l] += g[:, :l].sum(axis=1)
    if r:
        g[:, -r - 1] += g[:, -r:].sum(axis=1)
    return g[:, l : l + nx].copy()


def sponge_profile(n, before, after, strength):
    """1-D factor exp(-strength k^2) -- seisopt/wavesim.py:155-161."""
    prof = np.ones(n)
    kb = np.arange(before, 0, -1, dtype=np.float64)
    prof[:before] = np.exp(-strength * kb * kb)
    ka = np.arange(1, after + 1, dtype=np.float64)
    prof[n - after :] = np.exp(-strength * ka * ka)
    return prof


def bilinear_taps(points, dx, dz, pads, shape):
    """Rows, cols, weights (each (4, n)) -- seisopt/wavesim.py:168-180."""
    nzp, nxp = shape
    top, left = pads[0], pads[2]
    xf = np.array([p[0] for p in points]) / dx + left
    zf = np.array([p[1] for p in points]) / dz + top
    i0 = np.minimum(np.floor(zf).astype(int), nzp - 2)
    j0 = np.minimum(np.floor(xf).astype(int), nxp - 2)
    fz = zf - i0
    fx = xf - j0
    rows = np.stack([i0, i0 + 1, i0, i0 + 1])
    cols = np.stack([j0, j0, j0 + 1, j0 + 1])
    wts = np.stack([(1 - fz) * (1 - fx), fz * (1 - fx), (1 - fz) * fx, fz * fx])
    return rows, cols, wts


def cfl_limit(m_phys, dx, dz, safety, order=2):
    """Largest stable dt -- seisopt/wavesim.py:92-100 (x CFL8_FACTOR for order 8)."""
    c_max = float(1.0 / math.sqrt(np.min(m_phys)))
    bound = safety * min(dx, dz) / (c_max * math.sqrt(2.0))
    return bound * CFL8_FACTOR if order == 8 else bound


class Setup:
    """Per-model precompute, the oracle's counterpart of ``Workspace``
    (seisopt/wavesim.py:183-214)."""

    def __init__(self, m_phys, dx, dz, dt, sources, receivers, border=30,
                 strength=0.0053, cfl_safety=0.9, damp_top=True, order=2):
        m_phys = np.asarray(m_phys, dtype=np.float64)
        if order not in (2, 8):
            raise ValueError("order must be 2 or 8")
        bound = cfl_limit(m_phys, dx, dz, cfl_safety, order)
        if dt > bound:
            raise OracleStabilityError(f"dt={dt} exceeds stable bound {bound:.6g}")
        self.order = order
        self.nz, self.nx = m_phys.shape
        self.dx, self.dz, self.dt = float(dx), float(dz), float(dt)
        self.pads = pad_widths(border, damp_top)
        t, b, l, r = self.pads
        self.shape = (self.nz + t + b, self.nx + l + r)
        self.m_pad = extend_to_pad(m_phys, self.pads)
        self.inv_m = 1.0 / self.m_pad
        self.pz = sponge_profile(self.shape[0], t, b, strength)
        self.px = sponge_profile(self.shape[1], l, r, strength)
        self.damp = np.outer(self.pz, self.px)
        self.dt2 = self.dt * self.dt
        self.kx = 1.0 / (self.dx * self.dx)
        self.kz = 1.0 / (self.dz * self.dz)
        self.kc = -2.0 * (self.kx + self.kz)
        self.rec = bilinear_taps(receivers, dx, dz, self.pads, self.shape)
        self.src = bilinear_taps(sources, dx, dz, self.pads, self.shape)
        self.src_scale = 1.0 / (self.dx * self.dz)
        self.n_sources = len(sources)
        self.n_receivers = len(receivers)

    # -- spatial operator ---------------------------------------------------
    def lap(self, u, out):
        """Zero-exterior Laplacian.  order 2 follows seisopt/wavesim.py:216-223
        term by term; order 8 is the BASELINE substitution."""
        if self.order == 2:
            np.multiply(u, self.kc, out=out)
            out[1:, :] += u[:-1, :] * self.kz
            out[:-1, :] += u[1:, :] * self.kz
            out[:, 1:] += u[:, :-1] * self.kx
            out[:, :-1] += u[:, 1:] * self.kx
            return out
        np.multiply(u, LAP8[0] * (self.kz + self.kx), out=out)
        for k in range(1, 5):
            cz = LAP8[k] * self.kz
            out[k:, :] += u[:-k, :] * cz
            out[:-k, :] += u[k:, :] * cz
        for k in range(1, 5):
            cx = LAP8[k] * self.kx
            out[:, k:] += u[:, :-k] * cx
            out[:, :-k] += u[:, k:] * cx
        return out

    def sample(self, u):
        """Receiver sampling -- seisopt/wavesim.py:225-226."""
        rows, cols, w = self.rec
        return np.einsum("kr,kr->r", u[rows, cols], w)

    def inject(self, u, amps):
        """Receiver injection (duplicates add) -- seisopt/wavesim.py:228-229."""
        rows, cols, w = self.rec
        np.add.at(u, (rows, cols), w * amps)


# ---------------------------------------------------------------------------
# Time loops (seisopt/wavesim.py:259-346)
# ---------------------------------------------------------------------------


def forward_sweep(st: Setup, nt, amp=None, shot=0, grid_src=None, grid_scale=None,
                  keep=True):
    """Damped leapfrog from rest -- seisopt/wavesim.py:259-304.

    Returns (gather (nt, nrec), acceleration history (nt, nzp, nxp) or None).
    """
    u_now = np.zeros(st.shape)
    u_old = np.zeros(st.shape)  # already multiplied by the sponge
    work = np.empty(st.shape)
    traces = np.zeros((nt, st.n_receivers))
    hist = np.empty((nt, *st.shape)) if keep else None
    if amp is not None:
        sr = st.src[0][:, shot]
        sc = st.src[1][:, shot]
        sw = st.src[2][:, shot] * st.src_scale
    for n in range(nt):
        traces[n] = st.sample(u_now)
        st.lap(u_now, out=work)
        if grid_src is not None:
            work += grid_src[n] * grid_scale
        work *= st.inv_m
        if amp is not None and amp[n] != 0.0:
            np.add.at(work, (sr, sc), amp[n] * sw * st.inv_m[sr, sc])
        if keep:
            hist[n] = work
        # u_next = d (2 u - u_old + dt^2 a);  u_old <- d u
        work *= st.dt2
        work += u_now
        work += u_now
        work -= u_old
        work *= st.damp
        u_now *= st.damp
        u_old, u_now, work = u_now, work, u_old
    return traces, hist


def adjoint_sweep(st: Setup, ybar, image_against=None, keep_v=False):
    """Exact transpose of forward_sweep's data map -- seisopt/wavesim.py:307-346."""
    nt = ybar.shape[0]
    lam = np.zeros(st.shape)
    lam_old = np.zeros(st.shape)
    v = np.empty(st.shape)
    dl = np.empty(st.shape)
    nxt = np.empty(st.shape)
    image = np.zeros(st.shape) if image_against is not None else None
    v_hist = np.empty((nt, *st.shape)) if keep_v else None
    for n in range(nt - 1, -1, -1):
        np.multiply(st.damp, lam, out=dl)
        np.multiply(dl, st.inv_m, out=v)
        v *= st.dt2
        st.lap(v, out=nxt)
        nxt += dl
        nxt += dl
        lam_old *= st.damp
        nxt += lam_old
        st.inject(nxt, ybar[n])
        np.multiply(dl, -1.0, out=lam_old)
        lam, nxt = nxt, lam
        if image is not None:
            image -= image_against[n] * v
        if keep_v:
            v_hist[n] = v
    return image, v_hist


def field_energy(st: Setup, prev, cur):
    """Discrete leapfrog energy -- seisopt/wavesim.py:433-438."""
    vel = (cur - prev) / math.sqrt(st.dt2)
    kinetic = 0.5 * float(np.sum(st.m_pad * vel * vel))
    lap = st.lap(prev, out=np.empty_like(prev))
    return kinetic - 0.5 * float(np.sum(cur * lap))


# ---------------------------------------------------------------------------
# Objectives and gradients (seisopt/gradients.py)
# ---------------------------------------------------------------------------


def tree_sum(arrays):
    """Deterministic pairwise reduction -- seisopt/gradients.py:40-50."""
    items = [np.asarray(a) for a in arrays]
    if not items:
        raise ValueError("nothing to sum")
    while len(items) > 1:
        nxt = []
        for i in range(0, len(items), 2):
            nxt.append(items[i] + items[i + 1] if i + 1 < len(items) else items[i])
        items = nxt
    return items[0]


def trapezoid(nt):
    """seisopt/gradients.py:63-67."""
    w = np.ones(nt)
    w[0] = 0.5
    w[-1] = 0.5
    return w


def misfit_l2(synthetic, observed, dt):
    """Trapezoidal L2 misfit -- seisopt/gradients.py:70-79 (arrays (nt, nrec))."""
    if len(synthetic) != len(observed):
        raise ValueError("gather counts differ")
    total = 0.0
    for f, g in zip(synthetic, observed):
        if f.shape != g.shape:
            raise ValueError("gather shapes differ")
        d = f - g
        total += 0.5 * dt * float(np.einsum("t,tr->", trapezoid(f.shape[0]), d * d))
    return total


def _map(fn, n, threads):
    """Shot map in shot order -- seisopt/gradients.py:91-95."""
    if threads <= 1:
        return [fn(s) for s in range(n)]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(fn, range(n)))


def fwi_synthetic(st: Setup, wavelet, nt, threads=1, shots=None):
    """All-shot forward modelling -- seisopt/gradients.py:98-115."""
    ids = list(range(st.n_sources)) if shots is None else list(shots)
    return _map(lambda i: forward_sweep(st, nt, amp=wavelet, shot=ids[i], keep=False)[0],
                len(ids), threads)


def fwi_gradient(st: Setup, observed, wavelet, nt, threads=1, shots=None):
    """Misfit and exact gradient -- seisopt/gradients.py:118-155.

    Returns (value, grad (nz, nx), per-shot padded images)."""
    ids = list(range(st.n_sources)) if shots is None else list(shots)
    if len(observed) != len(ids):
        raise ValueError("observed data does not cover all sources")
    wq = trapezoid(nt)
    wdt = wq[:, None] * st.dt

    def one(i):
        traces, hist = forward_sweep(st, nt, amp=wavelet, shot=ids[i], keep=True)
        res = traces - observed[i]
        val = 0.5 * st.dt * float(np.einsum("t,tr->", wq, res * res))
        img, _ = adjoint_sweep(st, wdt * res, image_against=hist)
        return val, img

    out = _map(one, len(ids), threads)
    value = float(np.sum([o[0] for o in out]))
    grad = fold_pad(tree_sum([o[1] for o in out]), st.pads, st.nz, st.nx)
    return value, grad, [o[1] for o in out]


class BornOracle:
    """Born operator with cached background histories --
    seisopt/gradients.py:158-220."""

    def __init__(self, st: Setup, wavelet, nt, threads=1):
        self.st, self.nt, self.threads = st, nt, threads
        self.born_applies = 0
        self.adjoint_applies = 0
        self.histories = _map(
            lambda s: forward_sweep(st, nt, amp=wavelet, shot=s, keep=True)[1],
            st.n_sources, threads)

    def forward(self, m_r):
        scale = -extend_to_pad(np.asarray(m_r, dtype=np.float64), self.st.pads)
        out = _map(lambda s: forward_sweep(self.st, self.nt, grid_src=self.histories[s],
                                           grid_scale=scale, keep=False)[0],
                   self.st.n_sources, self.threads)
        self.born_applies += 1
        return out

    def adjoint(self, data):
        if len(data) != self.st.n_sources:
            raise ValueError("data does not cover all sources")
        imgs = _map(lambda s: adjoint_sweep(self.st, data[s],
                                            image_against=self.histories[s])[0],
                    self.st.n_sources, self.threads)
        self.adjoint_applies += 1
        return fold_pad(tree_sum(imgs), self.st.pads, self.st.nz, self.st.nx)


def lsrtm_objective(kernel: BornOracle, m_r, d_r):
    """J = 1/2 ||L m_r - d_r||^2 (no dt, no trapezoid) -- seisopt/gradients.py:253-277."""
    syn = kernel.forward(np.asarray(m_r, dtype=np.float64))
    res = [f - g for f, g in zip(syn, d_r)]
    value = 0.5 * sum(float(np.sum(r * r)) for r in res)
    return value, kernel.adjoint(res)


class Counters:
    """seisopt/counting.py:14-24."""

    def __init__(self):
        self.grad_evals = 0
        self.obj_evals = 0

    @property
    def grad_equivalents(self):
        return self.grad_evals + 0.5 * self.obj_evals


class FwiOracleObjective:
    """Objective protocol over flattened m -- seisopt/gradients.py:300-336."""

    def __init__(self, make_setup, observed, wavelet, nt, shape, threads=1):
        self.make_setup = make_setup  # m_phys -> Setup
        self.observed, self.wavelet, self.nt = observed, wavelet, nt
        self.shape, self.threads = shape, threads
        self.counters = Counters()

    def _m(self, p):
        m = np.asarray(p, dtype=np.float64).reshape(self.shape)
        if not np.all(np.isfinite(m)) or np.any(m <= 0):
            return None
        return m

    def value(self, p):
        m = self._m(p)
        if m is None:
            return float("inf")
        self.counters.obj_evals += 1
        st = self.make_setup(m)
        syn = fwi_synthetic(st, self.wavelet, self.nt, self.threads)
        return misfit_l2(syn, self.observed, st.dt)

    def value_and_grad(self, p):
        m = self._m(p)
        if m is None:
            raise ValueError("model is not positive and finite")
        st = self.make_setup(m)
        val, grad, _ = fwi_gradient(st, self.observed, self.wavelet, self.nt, self.threads)
        self.counters.grad_evals += 1
        return val, grad.ravel()


class LsrtmOracleObjective:
    """seisopt/gradients.py:339-378."""

    def __init__(self, kernel: BornOracle, d_r):
        self.kernel, self.d_r = kernel, d_r
        self.counters = Counters()

    def value(self, p):
        self.counters.obj_evals += 1
        st = self.kernel.st
        syn = self.kernel.forward(np.asarray(p, dtype=np.float64).reshape(st.nz, st.nx))
        return 0.5 * sum(float(np.sum((f - g) ** 2)) for f, g in zip(syn, self.d_r))

    def value_and_grad(self, p):
        st = self.kernel.st
        val, grad = lsrtm_objective(self.kernel, np.asarray(p).reshape(st.nz, st.nx), self.d_r)
        self.counters.grad_evals += 1
        return val, grad.ravel()


# ---------------------------------------------------------------------------
# Anderson acceleration (seisopt/optim/qr.py, seisopt/optim/anderson.py)
# ---------------------------------------------------------------------------

RANK_TOL = 1e-12  # seisopt/optim/anderson.py:22


class QRWindow:
    """Column-append / first-column-drop QR -- seisopt/optim/qr.py:22-104."""

    def __init__(self, rows):
        self.rows = rows
        self.q = np.zeros((rows, 0))
        self.r = np.zeros((0, 0))

    @property
    def ncols(self):
        return self.r.shape[1]

    def append(self, col):
        """CGS with one re-orthogonalisation -- qr.py:34-61."""
        a = np.asarray(col, dtype=np.float64)
        coef = self.q.T @ a
        resid = a - self.q @ coef
        corr = self.q.T @ resid
        resid -= self.q @ corr
        coef += corr
        rho = float(np.linalg.norm(resid))
        ref = max(float(np.linalg.norm(a)), 1.0)
        if rho <= 1e-300 or rho < 1e-15 * ref:
            qn, rho = np.zeros(self.rows), 0.0
        else:
            qn = resid / rho
        k = self.ncols
        self.q = np.column_stack([self.q, qn])
        grown = np.zeros((k + 1, k + 1))
        grown[:k, :k] = self.r
        grown[:k, k] = coef
        grown[k, k] = rho
        self.r = grown

    def drop_first(self):
        """Givens re-triangularisation -- qr.py:63-80."""
        k = self.ncols
        if k == 0:
            raise OracleEmptyWindow("drop on empty window")
        hess = np.ascontiguousarray(self.r[:, 1:])
        qq = self.q.copy()
        for i in range(k - 1):
            x, y = hess[i, i], hess[i + 1, i]
            h = math.hypot(x, y)
            c, s = (1.0, 0.0) if h == 0.0 else (x / h, y / h)
            rot = np.array([[c, s], [-s, c]])
            hess[i : i + 2, i:] = rot @ hess[i : i + 2, i:]
            qq[:, i : i + 2] = qq[:, i : i + 2] @ rot.T
        self.r = hess[: k - 1, :]
        self.q = qq[:, : k - 1]

    def solve(self, rhs):
        if self.ncols == 0:
            raise OracleEmptyWindow("solve on empty window")
        return solve_triangular(self.r, self.q.T @ rhs, lower=False)

    def residual_norm(self, rhs):
        rhs = np.asarray(rhs, dtype=np.float64)
        if self.ncols == 0:
            return float(np.linalg.norm(rhs))
        res = rhs - self.q @ (self.q.T @ rhs)
        return min(float(np.linalg.norm(res)), float(np.linalg.norm(rhs)))

    def diag(self):
        return np.abs(np.diag(self.r))

    def frobenius(self):
        return float(np.linalg.norm(self.r))


def recover_alpha(gamma):
    """gamma -> affine weights summing to one -- anderson.py:41-52."""
    m = len(gamma)
    a = np.empty(m + 1)
    a[0] = gamma[0]
    a[1:m] = gamma[1:] - gamma[:-1]
    a[m] = 1.0 - gamma[m - 1]
    for _ in range(3):
        gap = 1.0 - math.fsum(a)
        if gap == 0.0:
            break
        a[int(np.argmax(np.abs(a)))] += gap
    return a


class AAWindowOracle:
    """Sliding AA history -- seisopt/optim/anderson.py:55-112."""

    def __init__(self, dim, memory):
        if memory < 0:
            raise ValueError("memory must be non-negative")
        self.dim, self.memory = dim, memory
        self.qr = QRWindow(dim) if memory > 0 else None
        self.ps, self.gs, self.fs, self.dgs = [], [], [], []

    @property
    def m_k(self):
        return len(self.fs) - 1 if self.fs else 0

    @property
    def f_k(self):
        return self.fs[-1]

    def clear(self):
        self.__init__(self.dim, self.memory)

    def push(self, p, gval):
        p = np.asarray(p, dtype=np.float64)
        gval = np.asarray(gval, dtype=np.float64)
        f = gval - p
        if self.memory == 0:
            self.ps, self.gs, self.fs = [p], [gval], [f]
            return
        if self.fs:
            self.qr.append(f - self.fs[-1])
            self.dgs.append(gval - self.gs[-1])
        self.ps.append(p)
        self.gs.append(gval)
        self.fs.append(f)
        if self.qr.ncols > self.memory:
            self._drop()
        while self.qr.ncols > 0:  # safeguard, anderson.py:105-112
            if self.qr.diag().min() > RANK_TOL * max(self.qr.frobenius(), 1e-300):
                break
            self._drop()

    def _drop(self):
        self.qr.drop_first()
        for lst in (self.ps, self.gs, self.fs, self.dgs):
            lst.pop(0)


def aa_weights(win: AAWindowOracle):
    """(gamma, alpha, residual_norm) -- anderson.py:115-123."""
    if win.m_k == 0:
        raise OracleEmptyWindow("aa_weights needs at least one stored difference")
    gamma = win.qr.solve(win.f_k)
    return gamma, recover_alpha(gamma), win.qr.residual_norm(win.f_k)


def aa_step(win: AAWindowOracle, beta=1.0, weights=None):
    """anderson.py:126-148."""
    if not win.fs:
        raise OracleEmptyWindow("aa_step on an empty window")
    if win.m_k == 0:
        return win.gs[-1].copy()
    if weights is None:
        weights = aa_weights(win)
    gamma, alpha, _ = weights
    if beta == 1.0:
        out = win.gs[-1].copy()
        for gi, dg in zip(gamma, win.dgs):
            out -= gi * dg
        return out
    cp = sum(a * p for a, p in zip(alpha, win.ps))
    cg = sum(a * g for a, g in zip(alpha, win.gs))
    return (1.0 - beta) * cp + beta * cg


def default_eta(p0, g0):
    """seisopt/optim/problems.py:85-93."""
    ginf = float(np.max(np.abs(g0)))
    if ginf == 0.0:
        return 1.0
    scale = float(np.ptp(p0))
    if scale == 0.0:
        scale = max(1.0, float(np.max(np.abs(p0))))
    return 0.01 * scale / ginf


def _budget_ok(problem, budget, cost):
    """anderson.py:229-232."""
    return budget is None or problem.counters.grad_equivalents + cost <= budget + 1e-9


def blend_search(problem, jk, gk, pk, pbar, ptil, c1, max_bt, budget_ok):
    """Backtracking on the AA/SD blend -- anderson.py:356-376."""
    diff = ptil - pbar
    base = float(np.dot(gk, pbar - pk))
    cross = float(np.dot(gk, diff))
    lam = 1.0
    for _ in range(max_bt):
        if not budget_ok():
            return 0.0, pbar
        cand = pbar + lam * diff
        bound = jk + c1 * min(base + lam * cross, 0.0)
        trial = problem.value(cand)
        if np.isfinite(trial) and trial <= bound:
            return lam, cand
        lam *= 0.5
    return 0.0, pbar


def minimize_aa(problem, p0, memory, eta=None, budget=None, max_iters=None,
                grad_tol=0.0, c1=1e-4, max_backtracks=10):
    """Alg. 2 as implemented in anderson.py:283-353.

    Returns dict(p, rows=[(k, J, |g|, grad_evals, obj_evals, lambda)], eta,
    lambdas, inequality_log, iterates)."""
    p = np.asarray(p0, dtype=np.float64).copy()
    win = AAWindowOracle(p.size, memory)
    rows, lams, ineq, iterates = [], [], [], [p.copy()]
    k = 0
    while True:
        if not _budget_ok(problem, budget, 1.0):
            break
        val, g = problem.value_and_grad(p)
        if eta is None:
            eta = default_eta(p, g)
        gn = float(np.linalg.norm(g))
        done = (grad_tol and gn <= grad_tol) or (max_iters is not None and k >= max_iters)
        lam = 0.0
        if not done:
            pbar = p - eta * g
            win.push(p, pbar)
            if win.m_k == 0:
                pnext = pbar
            else:
                w = aa_weights(win)
                ineq.append((w[2], float(np.linalg.norm(win.f_k))))
                ptil = aa_step(win, weights=w)
                lam, pnext = blend_search(problem, val, g, p, pbar, ptil, c1, max_backtracks,
                                          lambda: _budget_ok(problem, budget, 0.5))
                if lam == 0.0:
                    win.clear()
                    pnext = pbar
            lams.append(lam)
        rows.append((k, val, gn, problem.counters.grad_evals, problem.counters.obj_evals, lam))
        if done:
            break
        p = pnext
        iterates.append(p.copy())
        k += 1
    return dict(p=p, rows=rows, eta=eta, lambdas=lams, inequality_log=ineq, iterates=iterates)


def armijo_search(value_fn, p, direction, grad_p, value_p, initial_step, c1, max_bt,
                  budget_ok=None):
    """Armijo backtracking -- seisopt/optim/linesearch.py:29-70.
    Returns (step, success)."""
    slope = float(np.dot(direction, grad_p))
    if slope >= 0.0 or initial_step <= 0.0:
        raise ValueError("not a descent direction / non-positive step")
    s = float(initial_step)
    for _ in range(max_bt):
        if budget_ok is not None and not budget_ok():
            return 0.0, False
        f = value_fn(p + s * direction)
        if np.isfinite(f) and f <= value_p + c1 * s * slope:
            return s, True
        s *= 0.5
    return 0.0, False


def minimize_sd(problem, p0, eta=None, max_iters=None, line_search=False, c1=1e-4,
                max_backtracks=10, budget=None):
    """Steepest descent -- anderson.py:235-280 (fixed step, or Armijo
    backtracking from eta with the eta * 0.5**max_backtracks fallback)."""
    p = np.asarray(p0, dtype=np.float64).copy()
    rows, k = [], 0
    while True:
        if not _budget_ok(problem, budget, 1.0):
            break
        val, g = problem.value_and_grad(p)
        if eta is None:
            eta = default_eta(p, g)
        gn = float(np.linalg.norm(g))
        done = max_iters is not None and k >= max_iters
        step = 0.0
        if not done:
            step = eta
            if line_search:
                s, ok = armijo_search(problem.value, p, -g, g, val, eta, c1, max_backtracks,
                                      lambda: _budget_ok(problem, budget, 0.5))
                step = s if ok else eta * 0.5 ** max_backtracks
        rows.append((k, val, gn, problem.counters.grad_evals, problem.counters.obj_evals, step))
        if done:
            break
        p = p - step * g
        k += 1
    return dict(p=p, rows=rows, eta=eta)


def aa_run(operator, p0, memory, iterations, beta=1.0, residual_tol=0.0):
    """Generic AA of a fixed-point operator -- anderson.py:168-203.
    Returns (iterates, residual_norms, combined_norms)."""
    p = np.asarray(p0, dtype=np.float64)
    win = AAWindowOracle(p.size, memory)
    its, res, comb = [p.copy()], [], []
    for _ in range(iterations):
        win.push(p, operator(p))
        fk = float(np.linalg.norm(win.f_k))
        if win.m_k == 0:
            pn, cn = aa_step(win, beta), fk
        else:
            w = aa_weights(win)
            pn, cn = aa_step(win, beta, w), w[2]
        its.append(pn)
        res.append(fk)
        comb.append(cn)
        p = pn
        if residual_tol and fk <= residual_tol:
            break
    return its, res, comb

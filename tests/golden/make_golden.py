"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``seisopt`` from /root/reference/pkg/src and writes small ``.npz``
fixtures next to this file.  The 8th-order fixtures use the one-method
substitution documented in SURVEY.md s0 item 1: ``Workspace.laplacian`` is
replaced by the 8th-order zero-exterior Laplacian and ``cfl_check`` is scaled
by sqrt(4/6.5016); everything else (time loop, taps, sponge, imaging, fold,
misfit, AA) is the reference's own code.  Library versions are recorded in
each fixture.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from seisopt import gradients as G  # noqa: E402
from seisopt import wavesim as W  # noqa: E402
from seisopt.grid import (AcquisitionGeometry, Grid2D, ReflectivityModel,  # noqa: E402
                          VelocityModel, make_ricker, smooth_model)
from seisopt.optim import anderson as A  # noqa: E402

from paper_2008_11778_b200 import synthetic  # noqa: E402  (input builders only)

_ORIG_LAP = W.Workspace.laplacian
_ORIG_CFL = W.cfl_check
C8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)
SYM8 = 205.0 / 72.0 + 2.0 * (8.0 / 5.0 + 1.0 / 5.0 + 8.0 / 315.0 + 1.0 / 560.0)


def _lap8(self, u, out):
    np.multiply(u, C8[0] * (self.rz + self.rx), out=out)
    for k in range(1, 5):
        c = C8[k] * self.rz
        out[k:, :] += u[:-k, :] * c
        out[:-k, :] += u[k:, :] * c
    for k in range(1, 5):
        c = C8[k] * self.rx
        out[:, k:] += u[:, :-k] * c
        out[:, :-k] += u[:, k:] * c
    return out


def _cfl8(model, dt=None, cfl_safety=1.0):
    return _ORIG_CFL(model, dt, cfl_safety) * math.sqrt(4.0 / SYM8)


def use_order(order):
    if order == 8:
        W.Workspace.laplacian = _lap8
        W.cfl_check = _cfl8
    else:
        W.Workspace.laplacian = _ORIG_LAP
        W.cfl_check = _ORIG_CFL


def versions():
    return dict(numpy=np.__version__, scipy=scipy.__version__)


def ref_types(case):
    """Rebuild a synthetic case with the reference's own types."""
    g = case["grid"]
    grid = Grid2D(nx=g.nx, nz=g.nz, dx=g.dx, dz=g.dz)
    geo = case["geometry"]
    geom = AcquisitionGeometry(geo.sources, geo.receivers, geo.dt, geo.nt)
    w = case["wavelet"]
    wav = make_ricker(w.peak_freq, geo.dt, geo.nt, t0=w.t0)
    cfg = W.SimConfig(border_width=case["config"].border_width)
    return grid, geom, wav, cfg


class Recorder:
    """Wraps an objective and records every model passed to value_and_grad
    (and the value and gradient the reference returned for it)."""

    def __init__(self, inner):
        self.inner = inner
        self.counters = inner.counters
        self.models = []
        self.values = []
        self.grads = []

    def value(self, p):
        return self.inner.value(p)

    def value_and_grad(self, p):
        self.models.append(np.array(p, copy=True))
        v, g = self.inner.value_and_grad(p)
        self.values.append(v)
        self.grads.append(np.array(g, copy=True))
        return v, g


def report_rows(res):
    return np.array([[r.iteration, r.objective, r.grad_norm, r.grad_evals, r.obj_evals,
                      r.step] for r in res.report.rows])


def make_c1(order, with_aa):
    use_order(order)
    case = synthetic.c1_case(order=order)
    grid, geom, wav, cfg = ref_types(case)
    true = VelocityModel(grid, case["true"].m)
    init = VelocityModel(grid, case["init"].m)
    obs = G.fwi_synthetic(true, wav, geom, cfg)
    ev = G.fwi_gradient(init, obs, wav, geom, cfg)
    out = dict(m_true=true.m, m_init=init.m, obs_shot2=obs[2].samples,
               value=ev.value, grad=ev.gradient, order=order, **versions())
    if with_aa:
        obj = Recorder(G.FwiObjective(grid, obs, wav, geom, cfg))
        res = A.minimize_aa(obj, init.m.ravel(), memory=5, max_iters=20)
        rows = np.array([[r.iteration, r.objective, r.grad_norm, r.grad_evals, r.obj_evals,
                          r.step] for r in res.report.rows])
        keep = [0, 1, 2, 5, 10, 19, 20]
        out.update(aa_rows=rows, aa_eta=res.extras["eta"], aa_keep=np.array(keep),
                   aa_iterates=np.stack([obj.models[k] for k in keep]),
                   aa_values=np.array([obj.values[k] for k in keep]),
                   aa_grads=np.stack([obj.grads[k] for k in keep]),
                   aa_final=res.p)
    np.savez_compressed(os.path.join(HERE, f"c1_o{order}.npz"), **out)


def small_setup(order, damp_top):
    grid = Grid2D(nx=60, nz=40, dx=20.0, dz=20.0)
    c = np.full(grid.shape, 1800.0)
    c[15:, :] = 2200.0
    c[28:, :] = 2600.0
    model = smooth_model(VelocityModel.from_velocity(grid, c), 3.0)
    sources = ((333.3, 0.0), (880.0, 47.5))
    # receivers: fractional positions, an exact duplicate, and the far edge
    # (x = extent_x clamps to j0 = nxp - 2 with tx = 1)
    receivers = tuple((x, 30.0) for x in np.linspace(0.0, 1180.0, 25)) + (
        (505.0, 37.5), (505.0, 37.5), (1180.0, 780.0))
    geom = AcquisitionGeometry(sources, receivers, dt=2e-3, nt=300)
    wav = make_ricker(12.0, 2e-3, 300, t0=0.08)
    cfg = W.SimConfig(border_width=10, damp_top=damp_top)
    return grid, model, geom, wav, cfg


def make_small(order, damp_top):
    use_order(order)
    grid, model, geom, wav, cfg = small_setup(order, damp_top)
    rng = np.random.default_rng(7)
    c_true = model.velocity.copy()
    c_true[18:24, 25:35] *= 1.06
    true = VelocityModel.from_velocity(grid, c_true)
    obs = G.fwi_synthetic(true, wav, geom, cfg)
    syn = G.fwi_synthetic(model, wav, geom, cfg)
    ev = G.fwi_gradient(model, obs, wav, geom, cfg)
    kern = G.BornKernel(model, wav, geom, cfg)
    m_r = rng.standard_normal(grid.shape) * 1e-8
    born = kern.forward(m_r)
    y = [W.ShotGather(s, rng.standard_normal((geom.nt, geom.n_receivers)), geom.dt)
         for s in range(geom.n_sources)]
    img = kern.adjoint(y)
    lev = G.lsrtm_objective(model, m_r * 0.5, born, kernel=kern)
    ws = W.Workspace(model, geom, cfg)
    tag = f"small_o{order}_{'top' if damp_top else 'free'}"
    np.savez_compressed(
        os.path.join(HERE, tag + ".npz"),
        m=model.m, m_true=true.m, obs=np.stack([o.samples for o in obs]),
        syn=np.stack([s.samples for s in syn]), value=ev.value, grad=ev.gradient,
        m_r=m_r, born=np.stack([b.samples for b in born]),
        y=np.stack([v.samples for v in y]), img=img, lsrtm_value=lev.value,
        lsrtm_grad=lev.gradient, rec_rows=ws.rec_rows, rec_cols=ws.rec_cols,
        rec_w=ws.rec_w, src_rows=ws.src_rows, src_cols=ws.src_cols, src_w=ws.src_w,
        damp=ws.damp, order=order, damp_top=damp_top, **versions())
    # AA trajectory on the small FWI problem (drives the reference optimizer)
    if order == 8 and damp_top:
        obj = Recorder(G.FwiObjective(grid, obs, wav, geom, cfg))
        res = A.minimize_aa(obj, model.m.ravel(), memory=3, max_iters=8)
        rows = np.array([[r.iteration, r.objective, r.grad_norm, r.grad_evals, r.obj_evals,
                          r.step] for r in res.report.rows])
        obj_sd = G.FwiObjective(grid, obs, wav, geom, cfg)
        sd = A.minimize_sd(obj_sd, model.m.ravel(), max_iters=3)
        np.savez_compressed(os.path.join(HERE, "aa_fwi_small.npz"), rows=rows,
                            eta=res.extras["eta"], iterates=np.stack(obj.models),
                            final=res.p, lambdas=np.array(res.extras["lambdas"]),
                            sd_final=sd.p, **versions())


def small_problem():
    """small_o8_top inputs through the reference: model, true model, observed."""
    use_order(8)
    grid, model, geom, wav, cfg = small_setup(8, True)
    c_true = model.velocity.copy()
    c_true[18:24, 25:35] *= 1.06
    true = VelocityModel.from_velocity(grid, c_true)
    obs = G.fwi_synthetic(true, wav, geom, cfg)
    return grid, model, geom, wav, cfg, obs


def make_solves():
    """Public single-shot solves (wavesim.py:354-430) on the small 8th-order
    case: forward_solve with history, born_solve (from the history and
    without), adjoint_solve.  Histories are stored as per-step norms plus a
    few whole planes (the full (nt, nzp, nxp) arrays are 10 MB each)."""
    grid, model, geom, wav, cfg, obs = small_problem()
    rng = np.random.default_rng(3)
    m_r = rng.standard_normal(grid.shape) * 1e-8
    refl = ReflectivityModel(grid, m_r)
    gat, hist = W.forward_solve(model, wav, geom, 1, cfg)
    gat_nohist, none = W.forward_solve(model, wav, geom, 0, cfg, keep_history=False)
    born_h = W.born_solve(model, refl, wav, geom, 1, cfg, background_history=hist)
    born0 = W.born_solve(model, refl, wav, geom, 0, cfg)
    ybar = W.ShotGather(0, rng.standard_normal((geom.nt, geom.n_receivers)), geom.dt)
    adj = W.adjoint_solve(model, ybar, geom, cfg)
    planes = np.array([10, 77, 150, 299])
    np.savez_compressed(
        os.path.join(HERE, "solves.npz"), m_r=m_r, gather1=gat.samples,
        gather0=gat_nohist.samples, hist_none=none is None,
        accel_norms=np.linalg.norm(hist.accel.reshape(geom.nt, -1), axis=1),
        accel_planes=hist.accel[planes], planes=planes,
        accel_phys=hist.accel_physical(150), born1=born_h.samples, born0=born0.samples,
        ybar=ybar.samples, v_norms=np.linalg.norm(adj.v.reshape(geom.nt, -1), axis=1),
        v_planes=adj.v[planes], **versions())


def make_lsrtm_objective():
    """LsrtmObjective (gradients.py:339-378) on the small case: value,
    value_and_grad, residual_norm, and the counters / kernel applies they
    leave (born_applies, adjoint_applies, grad_equivalents)."""
    grid, model, geom, wav, cfg, obs = small_problem()
    rng = np.random.default_rng(7)
    kern = G.BornKernel(model, wav, geom, cfg)
    m_true = rng.standard_normal(grid.shape) * 1e-8
    d_r = kern.forward(m_true)
    obj = G.LsrtmObjective(kern, d_r)
    p = (0.3 * m_true + 1e-9 * rng.standard_normal(grid.shape)).ravel()
    v = obj.value(p)
    vg, g = obj.value_and_grad(p)
    rn = obj.residual_norm(p)
    v0 = obj.value(np.zeros_like(p))
    np.savez_compressed(
        os.path.join(HERE, "lsrtm_objective.npz"), m_true=m_true, p=p, value=v,
        vg_value=vg, grad=g, residual_norm=rn, value0=v0,
        d_r=np.stack([d.samples for d in d_r]),
        counters=np.array([obj.counters.grad_evals, obj.counters.obj_evals]),
        applies=np.array([kern.born_applies, kern.adjoint_applies, kern.grad_equivalents]),
        **versions())
    # restarted GMRES on the normal equations (krylov.py:224-258), both starts
    from seisopt import krylov as K
    out = {}
    for tag, restart, iters, zero in (("rtm", 3, 9, False), ("zero", 5, 15, True)):
        kk = G.BornKernel(model, wav, geom, cfg)
        x, res = K.lsrtm_gmres(model, d_r, wav, geom, cfg, restart=restart, iterations=iters,
                               zero_start=zero, kernel=kk)
        out[f"{tag}_x"] = x
        out[f"{tag}_hist"] = np.array([[h.outer_iter, h.inner_iter, h.residual_norm,
                                        h.grad_equivalents] for h in res.history])
        out[f"{tag}_converged"] = res.converged
        out[f"{tag}_applies"] = np.array([kk.born_applies, kk.adjoint_applies])
    np.savez_compressed(os.path.join(HERE, "lsrtm_gmres.npz"), d_r=np.stack([d.samples for d in d_r]),
                        **out, **versions())


def make_quasi_newton():
    """minimize_lbfgs / minimize_ncg (optim/quasi_newton.py:123-208) on the
    small FWI problem, and the gradient-equivalent budget veto
    (optim/anderson.py:229-232) of minimize_aa / minimize_sd / minimize_lbfgs."""
    from seisopt.optim import quasi_newton as QN
    grid, model, geom, wav, cfg, obs = small_problem()
    out = {}
    res = QN.minimize_lbfgs(G.FwiObjective(grid, obs, wav, geom, cfg), model.m.ravel(),
                            memory=3, max_iters=4)
    out.update(lbfgs_rows=report_rows(res), lbfgs_final=res.p, lbfgs_eta=res.extras["eta"])
    res = QN.minimize_ncg(G.FwiObjective(grid, obs, wav, geom, cfg), model.m.ravel(),
                          max_iters=3)
    out.update(ncg_rows=report_rows(res), ncg_final=res.p)
    # budget veto: stops on grad_equivalents + cost > budget
    for tag, fn in (("aa", lambda o: A.minimize_aa(o, model.m.ravel(), memory=3, budget=5.5)),
                    ("sd", lambda o: A.minimize_sd(o, model.m.ravel(), budget=3.0,
                                                   line_search=True)),
                    ("lbfgs", lambda o: QN.minimize_lbfgs(o, model.m.ravel(), memory=3,
                                                          budget=4.5))):
        o = G.FwiObjective(grid, obs, wav, geom, cfg)
        r = fn(o)
        out[f"budget_{tag}_rows"] = report_rows(r)
        out[f"budget_{tag}_final"] = r.p
        out[f"budget_{tag}_counters"] = np.array([o.counters.grad_evals, o.counters.obj_evals])
    np.savez_compressed(os.path.join(HERE, "quasi_newton.npz"), **out, **versions())


def make_aa_window():
    """Window sequence with a full window, drops and a dependent column."""
    use_order(2)
    rng = np.random.default_rng(11)
    n, memory = 500, 4
    win = A.AAWindow(n, memory)
    basis = rng.standard_normal((n, 3))
    ps, gs, recs = [], [], []
    for k in range(12):
        p = rng.standard_normal(n) + basis @ rng.standard_normal(3)
        g = rng.standard_normal(n) + basis @ rng.standard_normal(3)
        if k == 7:  # make f_7 - f_6 parallel to f_6 - f_5 -> dependent column
            f5 = gs[5] - ps[5]
            f6 = gs[6] - ps[6]
            g = p + f6 + 2.0 * (f6 - f5)
        ps.append(p)
        gs.append(g)
        win.push(p, g)
        rec = dict(m_k=win.m_k)
        if win.m_k > 0:
            w = A.aa_weights(win)
            gamma = np.zeros(memory)
            alpha = np.zeros(memory + 1)
            gamma[: len(w.gamma)] = w.gamma
            alpha[: len(w.alpha)] = w.alpha
            rec.update(gamma=gamma, alpha=alpha, resid=w.residual_norm,
                       step1=A.aa_step(win, 1.0, w), step_half=A.aa_step(win, 0.5, w))
        else:
            rec.update(gamma=np.zeros(memory), alpha=np.zeros(memory + 1), resid=np.nan,
                       step1=A.aa_step(win), step_half=A.aa_step(win, 0.5))
        recs.append(rec)
    np.savez_compressed(
        os.path.join(HERE, "aa_window.npz"), n=n, memory=memory, ps=np.stack(ps),
        gs=np.stack(gs), m_k=np.array([r["m_k"] for r in recs]),
        gamma=np.stack([r["gamma"] for r in recs]), alpha=np.stack([r["alpha"] for r in recs]),
        resid=np.array([r["resid"] for r in recs]), step1=np.stack([r["step1"] for r in recs]),
        step_half=np.stack([r["step_half"] for r in recs]), **versions())


def make_aa_illcond():
    """Window sequence with nearly dependent residual differences
    (rho / ||a|| = 1e-6 .. 1e-9: below what a Gram / Cholesky solve resolves,
    above the 1e-12 rank safeguard) and one the safeguard sheds (1e-14)."""
    use_order(2)
    rng = np.random.default_rng(23)
    n, memory = 400, 5
    win = A.AAWindow(n, memory)
    ps, gs, recs = [], [], []
    eps = {4: 1e-6, 6: 1e-8, 8: 1e-9, 10: 1e-14, 12: 1e-7}
    for k in range(14):
        p = rng.standard_normal(n)
        g = rng.standard_normal(n)
        if k in eps and k >= 2:
            f1 = gs[k - 1] - ps[k - 1]
            f2 = gs[k - 2] - ps[k - 2]
            d = f1 - f2
            noise = rng.standard_normal(n)
            noise *= eps[k] * np.linalg.norm(d) / np.linalg.norm(noise)
            g = p + f1 + 0.7 * d + noise  # f_k - f_{k-1} = 0.7 (f_{k-1} - f_{k-2}) + noise
        ps.append(p)
        gs.append(g)
        win.push(p, g)
        rec = dict(m_k=win.m_k)
        w = A.aa_weights(win) if win.m_k > 0 else None
        gamma = np.zeros(memory)
        if w is not None:
            gamma[: len(w.gamma)] = w.gamma
        rec.update(gamma=gamma, resid=w.residual_norm if w is not None else np.nan,
                   step1=A.aa_step(win, 1.0, w) if w is not None else A.aa_step(win),
                   diag=np.pad(win.qr.diag(), (0, memory - win.qr.ncols)))
        recs.append(rec)
    np.savez_compressed(
        os.path.join(HERE, "aa_illcond.npz"), n=n, memory=memory, ps=np.stack(ps),
        gs=np.stack(gs), m_k=np.array([r["m_k"] for r in recs]),
        gamma=np.stack([r["gamma"] for r in recs]), resid=np.array([r["resid"] for r in recs]),
        step1=np.stack([r["step1"] for r in recs]), diag=np.stack([r["diag"] for r in recs]),
        **versions())


def make_aa_run():
    """aa_run on a contractive affine fixed point G(p) = M p + c (beta 1 and
    0.7), and Armijo steepest descent on the small FWI problem."""
    use_order(2)
    rng = np.random.default_rng(5)
    n = 120
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    mat = q @ np.diag(np.linspace(-0.9, 0.95, n)) @ q.T
    c = rng.standard_normal(n)
    p0 = rng.standard_normal(n)
    out = dict(n=n, mat=mat, c=c, p0=p0)
    for tag, memory, beta, iters in (("b1", 5, 1.0, 14), ("b07", 3, 0.7, 12), ("m0", 0, 1.0, 6)):
        tr = A.aa_run(lambda p: mat @ p + c, p0, memory, iters, beta=beta)
        out[f"{tag}_iterates"] = np.stack(tr.iterates)
        out[f"{tag}_res"] = np.array(tr.residual_norms)
        out[f"{tag}_comb"] = np.array(tr.combined_norms)
    tr = A.aa_run(lambda p: mat @ p + c, p0, 4, 40, residual_tol=0.05)
    out["tol_iterates"] = np.stack(tr.iterates)
    np.savez_compressed(os.path.join(HERE, "aa_run.npz"), **out, **versions())
    # steepest descent with the Armijo search (minimize_sd(line_search=True))
    use_order(8)
    grid, model, geom, wav, cfg = small_setup(8, True)
    c_true = model.velocity.copy()
    c_true[18:24, 25:35] *= 1.06
    obs = G.fwi_synthetic(VelocityModel.from_velocity(grid, c_true), wav, geom, cfg)
    res = A.minimize_sd(G.FwiObjective(grid, obs, wav, geom, cfg), model.m.ravel(),
                        eta=None, max_iters=3, line_search=True)
    rows = np.array([[r.iteration, r.objective, r.grad_norm, r.grad_evals, r.obj_evals,
                      r.step] for r in res.report.rows])
    big = A.minimize_sd(G.FwiObjective(grid, obs, wav, geom, cfg), model.m.ravel(),
                        eta=6.0 * res.extras["eta"], max_iters=2, line_search=True,
                        max_backtracks=2)
    big_rows = np.array([[r.iteration, r.objective, r.grad_norm, r.grad_evals, r.obj_evals,
                          r.step] for r in big.report.rows])
    np.savez_compressed(os.path.join(HERE, "sd_linesearch.npz"), rows=rows, final=res.p,
                        eta=res.extras["eta"], big_rows=big_rows, big_final=big.p,
                        **versions())


def make_c3(threads=6):
    """The benched workload itself (BASELINE configs[2], C3): the full 30-shot,
    nt 4000 FWI gradient of the reference (`gradients.py:118-155`) at the
    smoothed initial model, observed data synthesised by the reference from
    the seeded layered-fault true model (`gradients.py:98-115`), 8th order.
    The 30 x 4000 x 601 observed gathers (577 MB) are not stored: the fixture
    keeps per-shot norms and a few full traces of them (and of the synthetic
    at the initial model) so a GPU test can pin its own synthesis first."""
    use_order(8)
    case = synthetic.layered_case("c3")
    grid, geom, wav, cfg = ref_types(case)
    true = VelocityModel(grid, case["true"].m)
    init = VelocityModel(grid, case["init"].m)
    obs = G.fwi_synthetic(true, wav, geom, cfg, threads=threads)
    syn = G.fwi_synthetic(init, wav, geom, cfg, threads=threads)
    ev = G.fwi_gradient(init, obs, wav, geom, cfg, threads=threads)
    shot_misfit = np.array([G.misfit_l2([s], [o]) for s, o in zip(syn, obs)])
    trace_shots = np.array([0, 11, 29])
    trace_recs = np.array([0, 300, 600])
    np.savez_compressed(
        os.path.join(HERE, "c3_full.npz"),
        m_init=init.m, m_true_sum=float(np.sum(true.m)), value=ev.value, grad=ev.gradient,
        obs_norm=np.array([np.linalg.norm(o.samples) for o in obs]),
        syn_norm=np.array([np.linalg.norm(s.samples) for s in syn]),
        shot_misfit=shot_misfit, trace_shots=trace_shots, trace_recs=trace_recs,
        obs_traces=np.stack([obs[s].samples[:, trace_recs] for s in trace_shots]),
        syn_traces=np.stack([syn[s].samples[:, trace_recs] for s in trace_shots]),
        order=8, **versions())


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    make_aa_window()
    make_aa_illcond()
    make_aa_run()
    for order in (2, 8):
        for top in (True, False):
            make_small(order, top)
    make_c1(2, with_aa=False)
    make_c1(8, with_aa=True)
    print("goldens written to", HERE)

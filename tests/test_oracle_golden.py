"""Pin the CPU oracle against golden vectors from the unmodified reference.

The fixtures in tests/golden were produced by tests/golden/make_golden.py,
which runs seisopt itself (2nd order) or seisopt with the one-method 8th-order
Laplacian substitution.  The oracle must reproduce them to round-off; in
practice it is bit-identical because it follows the reference's operation
order.
"""

import numpy as np
import pytest

import oracle
from cases import c1, golden, oracle_setup, rel, small_case

TOL = 1e-13


@pytest.mark.parametrize("order", [2, 8])
@pytest.mark.parametrize("damp_top", [True, False])
def test_small_case(order, damp_top):
    case = small_case(order, damp_top)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st = oracle_setup(g["m"], grid, geom, cfg)
    # bilinear taps and sponge: exact
    for mine, name in zip(st.rec, ("rec_rows", "rec_cols", "rec_w")):
        assert np.array_equal(mine, g[name])
    for mine, name in zip(st.src, ("src_rows", "src_cols", "src_w")):
        assert np.array_equal(mine, g[name])
    assert np.array_equal(st.damp, g["damp"])
    st_true = oracle_setup(g["m_true"], grid, geom, cfg)
    obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt)
    assert rel(np.stack(obs), g["obs"]) <= TOL
    syn = oracle.fwi_synthetic(st, wav.samples, geom.nt)
    assert rel(np.stack(syn), g["syn"]) <= TOL
    val, grad, _ = oracle.fwi_gradient(st, list(g["obs"]), wav.samples, geom.nt)
    assert abs(val - float(g["value"])) <= TOL * abs(float(g["value"]))
    assert rel(grad, g["grad"]) <= TOL
    born = oracle.BornOracle(st, wav.samples, geom.nt)
    d = born.forward(g["m_r"])
    assert rel(np.stack(d), g["born"]) <= TOL
    img = born.adjoint(list(g["y"]))
    assert rel(img, g["img"]) <= TOL
    lval, lgrad = oracle.lsrtm_objective(born, g["m_r"] * 0.5, list(g["born"]))
    assert abs(lval - float(g["lsrtm_value"])) <= TOL * abs(float(g["lsrtm_value"]))
    assert rel(lgrad, g["lsrtm_grad"]) <= TOL


@pytest.mark.parametrize("order", [2, 8])
def test_c1_gradient(order):
    case = c1(order)
    g = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st_true = oracle_setup(g["m_true"], grid, geom, cfg)
    obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt, threads=5)
    assert rel(obs[2], g["obs_shot2"]) <= TOL
    st = oracle_setup(g["m_init"], grid, geom, cfg)
    val, grad, _ = oracle.fwi_gradient(st, obs, wav.samples, geom.nt, threads=5)
    assert abs(val - float(g["value"])) <= TOL * float(g["value"])
    assert rel(grad, g["grad"]) <= TOL


def test_aa_window_sequence():
    g = golden("aa_window")
    n, memory = int(g["n"]), int(g["memory"])
    win = oracle.AAWindowOracle(n, memory)
    for k in range(len(g["ps"])):
        win.push(g["ps"][k], g["gs"][k])
        assert win.m_k == int(g["m_k"][k])
        if win.m_k:
            w = oracle.aa_weights(win)
            assert np.allclose(w[0], g["gamma"][k][: win.m_k], rtol=1e-12, atol=1e-12)
            assert np.array_equal(w[1], g["alpha"][k][: win.m_k + 1]) or np.allclose(
                w[1], g["alpha"][k][: win.m_k + 1], rtol=1e-12, atol=1e-12)
            assert abs(w[2] - g["resid"][k]) <= 1e-12 * max(1.0, abs(g["resid"][k]))
            assert rel(oracle.aa_step(win, 1.0, w), g["step1"][k]) <= 1e-13
            assert rel(oracle.aa_step(win, 0.5, w), g["step_half"][k]) <= 1e-13
        else:
            assert rel(oracle.aa_step(win), g["step1"][k]) == 0.0
    # the dependent column pushed at k=7 must have shrunk the window
    assert int(g["m_k"][7]) < min(7, memory)



def test_aa_illcond_sequence():
    """Oracle QR window vs the reference on nearly dependent differences
    (tests/golden/make_golden.py:make_aa_illcond): same window sizes, R
    diagonals and weights to the conditioning of the window."""
    g = golden("aa_illcond")
    n, memory = int(g["n"]), int(g["memory"])
    win = oracle.AAWindowOracle(n, memory)
    for k in range(len(g["ps"])):
        win.push(g["ps"][k], g["gs"][k])
        assert win.m_k == int(g["m_k"][k]), k
        if win.m_k:
            w = oracle.aa_weights(win)
            assert rel(w[0], g["gamma"][k][: win.m_k]) <= 1e-9
            assert rel(oracle.aa_step(win, 1.0, w), g["step1"][k]) <= 1e-9
    # the 1e-14-dependent difference pushed at k=10 triggered the safeguard
    assert int(g["m_k"][10]) == 1

def test_aa_fwi_trajectory():
    g = golden("aa_fwi_small")
    case = small_case(8, True)
    gs = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]

    def make(m):
        return oracle_setup(m, grid, geom, cfg)

    obj = oracle.FwiOracleObjective(make, list(gs["obs"]), wav.samples, geom.nt, grid.shape)
    res = oracle.minimize_aa(obj, gs["m"].ravel(), memory=3, max_iters=8)
    rows = np.array(res["rows"])
    assert rows.shape == g["rows"].shape
    assert np.array_equal(rows[:, [0, 3, 4]], g["rows"][:, [0, 3, 4]])
    assert np.allclose(rows[:, 1], g["rows"][:, 1], rtol=1e-12)
    assert np.array_equal(rows[:, 5], g["rows"][:, 5])
    assert rel(res["p"], g["final"]) <= 1e-12
    assert abs(res["eta"] - float(g["eta"])) <= 1e-15 * float(g["eta"])
    # AA(0) == steepest descent
    obj0 = oracle.FwiOracleObjective(make, list(gs["obs"]), wav.samples, geom.nt, grid.shape)
    r0 = oracle.minimize_aa(obj0, gs["m"].ravel(), memory=0, max_iters=3)
    assert rel(r0["p"], g["sd_final"]) == 0.0


def test_aa_run_fixed_point():
    """Generic fixed-point AA (anderson.py:168-203) against the reference run."""
    g = golden("aa_run")
    mat, c = g["mat"], g["c"]

    def op(p):
        return mat @ p + c

    for tag, memory, beta, iters in (("b1", 5, 1.0, 14), ("b07", 3, 0.7, 12), ("m0", 0, 1.0, 6)):
        its, res, comb = oracle.aa_run(op, g["p0"], memory, iters, beta=beta)
        assert rel(np.stack(its), g[f"{tag}_iterates"]) <= 1e-13
        assert np.allclose(res, g[f"{tag}_res"], rtol=1e-13)
        assert np.allclose(comb, g[f"{tag}_comb"], rtol=1e-12)
        # the combined residual never exceeds the plain one
        assert all(cn <= fk * (1 + 1e-12) for cn, fk in zip(comb, res))
    its, _, _ = oracle.aa_run(op, g["p0"], 4, 40, residual_tol=0.05)
    assert len(its) == len(g["tol_iterates"])
    assert rel(np.stack(its), g["tol_iterates"]) <= 1e-13


def test_sd_armijo_trajectory():
    """minimize_sd(line_search=True) (anderson.py:235-280 + linesearch.py:29-70)."""
    g = golden("sd_linesearch")
    case = small_case(8, True)
    gs = case["gold"]
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]

    def make(m):
        return oracle_setup(m, grid, geom, cfg)

    obs = oracle.fwi_synthetic(make(gs["m_true"]), wav.samples, geom.nt)
    obj = oracle.FwiOracleObjective(make, obs, wav.samples, geom.nt, grid.shape)
    res = oracle.minimize_sd(obj, gs["m"].ravel(), max_iters=3, line_search=True)
    rows = np.array(res["rows"])
    assert np.array_equal(rows[:, [0, 3, 4]], g["rows"][:, [0, 3, 4]])
    assert np.allclose(rows[:, [1, 2, 5]], g["rows"][:, [1, 2, 5]], rtol=1e-12)
    assert rel(res["p"], g["final"]) <= 1e-12
    obj = oracle.FwiOracleObjective(make, obs, wav.samples, geom.nt, grid.shape)
    big = oracle.minimize_sd(obj, gs["m"].ravel(), eta=6.0 * float(g["eta"]), max_iters=2,
                             line_search=True, max_backtracks=2)
    rows = np.array(big["rows"])
    assert np.array_equal(rows[:, [0, 3, 4]], g["big_rows"][:, [0, 3, 4]])
    assert np.allclose(rows[:, [1, 2, 5]], g["big_rows"][:, [1, 2, 5]], rtol=1e-12)
    assert rel(big["p"], g["big_final"]) <= 1e-12


# ---------------------------------------------------------------------------
# round-2 fixtures: the oracle must reproduce them as well
# ---------------------------------------------------------------------------


def test_c3_full_fixture_one_shot():
    """Shot 11 of the benched C3 workload (201 x 601, nt 4000, 8th order):
    the oracle's synthesis of the true and initial models reproduces the
    reference's per-shot norms, traces and misfit (c3_full.npz)."""
    from paper_2008_11778_b200 import synthetic
    g = golden("c3_full")
    case = synthetic.layered_case("c3")
    assert rel(case["init"].m, g["m_init"]) <= 1e-14
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    s = 11
    ts = list(g["trace_shots"])
    k = ts.index(s)
    out = []
    for m in (case["true"].m, case["init"].m):
        st = oracle_setup(m, grid, geom, cfg)
        tr, _ = oracle.forward_sweep(st, geom.nt, amp=wav.samples, shot=s, keep=False)
        out.append(tr)
    obs, syn = out
    assert abs(np.linalg.norm(obs) - g["obs_norm"][s]) <= TOL * g["obs_norm"][s]
    assert abs(np.linalg.norm(syn) - g["syn_norm"][s]) <= TOL * g["syn_norm"][s]
    assert rel(obs[:, g["trace_recs"]], g["obs_traces"][k]) <= TOL
    assert rel(syn[:, g["trace_recs"]], g["syn_traces"][k]) <= TOL
    mis = oracle.misfit_l2([syn], [obs], geom.dt)
    assert abs(mis - g["shot_misfit"][s]) <= 1e-12 * g["shot_misfit"][s]


def test_solves_fixture():
    """forward_solve / born_solve / adjoint_solve (wavesim.py:354-430)."""
    g = golden("solves")
    case = small_case(8, True)
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st = oracle_setup(case["gold"]["m"], grid, geom, cfg)
    tr, hist = oracle.forward_sweep(st, geom.nt, amp=wav.samples, shot=1, keep=True)
    assert rel(tr, g["gather1"]) <= TOL
    assert rel(np.linalg.norm(hist.reshape(geom.nt, -1), axis=1), g["accel_norms"]) <= TOL
    assert rel(hist[g["planes"]], g["accel_planes"]) <= TOL
    scale = -oracle.extend_to_pad(g["m_r"], st.pads)
    born1, _ = oracle.forward_sweep(st, geom.nt, grid_src=hist, grid_scale=scale, keep=False)
    assert rel(born1, g["born1"]) <= TOL
    _, vh = oracle.adjoint_sweep(st, g["ybar"], keep_v=True)
    assert rel(np.linalg.norm(vh.reshape(geom.nt, -1), axis=1), g["v_norms"]) <= TOL
    assert rel(vh[g["planes"]], g["v_planes"]) <= TOL


def test_lsrtm_objective_fixture():
    """LsrtmObjective value / gradient / residual norm (gradients.py:339-378)."""
    g = golden("lsrtm_objective")
    case = small_case(8, True)
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    st = oracle_setup(case["gold"]["m"], grid, geom, cfg)
    born = oracle.BornOracle(st, wav.samples, geom.nt)
    assert rel(np.stack(born.forward(g["m_true"])), g["d_r"]) <= TOL
    obj = oracle.LsrtmOracleObjective(born, list(g["d_r"]))
    v = obj.value(g["p"])
    vg, grad = obj.value_and_grad(g["p"])
    assert abs(v - float(g["value"])) <= TOL * float(g["value"])
    assert abs(vg - float(g["vg_value"])) <= TOL * float(g["vg_value"])
    assert rel(grad, g["grad"]) <= TOL


def test_budget_fixture_minimize_aa():
    """minimize_aa's gradient-equivalent budget veto (anderson.py:229-232)."""
    g = golden("quasi_newton")
    case = small_case(8, True)
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    obs = list(case["gold"]["obs"])
    obj = oracle.FwiOracleObjective(lambda m: oracle_setup(m, grid, geom, cfg), obs,
                                    wav.samples, geom.nt, (grid.nz, grid.nx))
    res = oracle.minimize_aa(obj, case["gold"]["m"].ravel(), memory=3, budget=5.5)
    rows = np.asarray(res["rows"], dtype=np.float64)
    assert rel(res["p"], g["budget_aa_final"]) <= 1e-12
    ref = g["budget_aa_rows"]
    assert rows.shape == ref.shape
    assert np.array_equal(rows[:, [0, 3, 4]], ref[:, [0, 3, 4]])
    assert np.allclose(rows[:, 1], ref[:, 1], rtol=1e-12)

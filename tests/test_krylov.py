"""Restarted GMRES restatement vs the reference's (CPU, torch CPU tensors) and
the LSRTM normal-equations solve on the GPU."""

import sys

import numpy as np
import pytest
import torch

from paper_2008_11778_b200 import krylov


def _system(n, seed):
    rng = np.random.default_rng(seed)
    a = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    return a, rng.standard_normal(n)


def test_gmres_solves_and_is_monotone():
    a, b = _system(12, 0)
    op = krylov.LinearOperator.from_matrix(a)
    res = krylov.gmres_restarted(op, b, restart=12, tol=1e-12, max_outer=3)
    assert res.converged
    x = res.x.numpy()
    assert np.linalg.norm(a @ x - b) <= 1e-10 * np.linalg.norm(b)
    r = res.residual_norms()
    assert np.all(np.diff(r[1:]) <= 1e-12 * r[0])
    with pytest.raises(ValueError):
        krylov.gmres_restarted(op, b, restart=0)


@pytest.mark.parametrize("restart,iters", [(3, 9), (5, 20), (20, 8)])
def test_gmres_matches_reference(restart, iters, reference_available):
    if not reference_available:
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from seisopt import krylov as rk
    a, b = _system(16, restart)
    ref = rk.gmres_restarted(rk.LinearOperator.from_matrix(a), b, restart=restart, tol=1e-14,
                             max_outer=5, cost_per_matvec=1.0, cost_offset=0.5,
                             max_total_inner=iters)
    mine = krylov.gmres_restarted(krylov.LinearOperator.from_matrix(a), b, restart=restart,
                                  tol=1e-14, max_outer=5, cost_per_matvec=1.0, cost_offset=0.5,
                                  max_total_inner=iters)
    assert [(h.outer_iter, h.inner_iter) for h in ref.history] == \
        [(h.outer_iter, h.inner_iter) for h in mine.history]
    assert np.allclose(ref.residual_norms(), mine.residual_norms(), rtol=1e-9, atol=1e-14)
    assert [h.grad_equivalents for h in ref.history] == [h.grad_equivalents for h in mine.history]
    assert np.allclose(ref.x, mine.x.numpy(), rtol=1e-9, atol=1e-12)
    assert ref.converged == mine.converged


@pytest.mark.gpu
def test_lsrtm_gmres_on_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from cases import small_case
    from paper_2008_11778_b200 import gradients
    case = small_case(8, True)
    g = case["gold"]
    from paper_2008_11778_b200.model import VelocityModel
    bg = VelocityModel(case["grid"], g["m"])
    kern = gradients.BornKernel(bg, case["wavelet"], case["geometry"], case["config"])
    m_r, res = krylov.lsrtm_gmres(bg, list(g["born"]), case["wavelet"], case["geometry"],
                                  case["config"], restart=3, iterations=9, kernel=kern)
    r = res.residual_norms()
    assert r[-1] < 0.2 * r[0]
    assert np.all(np.isfinite(m_r))
    # from zero, the normal-equation solution fits the Born data of the true m_r
    m0, res0 = krylov.lsrtm_gmres(bg, list(g["born"]), case["wavelet"], case["geometry"],
                                  case["config"], restart=5, iterations=15, zero_start=True,
                                  kernel=kern)
    d_fit = kern.forward(m0)
    err = np.linalg.norm(np.stack([x.samples for x in d_fit]) - g["born"]) / np.linalg.norm(g["born"])
    assert err < 0.5

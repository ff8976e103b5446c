"""L-BFGS / nCG restatements vs the reference's on quadratic problems (CPU,
torch CPU tensors), and on the GPU FWI objective."""

import sys

import numpy as np
import pytest
import torch

from paper_2008_11778_b200 import quasi_newton as qn
from paper_2008_11778_b200.model import EvalCounters


class TorchQuadratic:
    """J(p) = 1/2 p^T A p - b^T p on torch tensors (test fixture)."""

    def __init__(self, a, b):
        self.a = torch.as_tensor(a)
        self.b = torch.as_tensor(b)
        self.counters = EvalCounters()

    def value(self, p):
        self.counters.obj_evals += 1
        return float(0.5 * p @ self.a @ p - self.b @ p)

    def value_and_grad(self, p):
        self.counters.grad_evals += 1
        return float(0.5 * p @ self.a @ p - self.b @ p), self.a @ p - self.b


def _problem(n=8, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, n))
    a = q @ q.T + n * np.eye(n)
    return a, rng.standard_normal(n), rng.standard_normal(n)


@pytest.mark.parametrize("method", ["lbfgs", "ncg"])
def test_matches_reference_trajectory(method, reference_available):
    if not reference_available:
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from seisopt.optim import problems, quasi_newton as rqn
    a, b, p0 = _problem()
    ref_obj = problems.QuadraticObjective(a, b)
    mine_obj = TorchQuadratic(a, b)
    if method == "lbfgs":
        ref = rqn.minimize_lbfgs(ref_obj, p0, memory=3, max_iters=12)
        mine = qn.minimize_lbfgs(mine_obj, torch.as_tensor(p0), memory=3, max_iters=12)
    else:
        ref = rqn.minimize_ncg(ref_obj, p0, max_iters=12)
        mine = qn.minimize_ncg(mine_obj, torch.as_tensor(p0), max_iters=12)
    rr = [(r.iteration, r.grad_evals, r.obj_evals) for r in ref.report.rows]
    mr = [(r.iteration, r.grad_evals, r.obj_evals) for r in mine.report.rows]
    assert rr == mr
    assert np.allclose([r.objective for r in ref.report.rows],
                       [r.objective for r in mine.report.rows], rtol=1e-10)
    assert np.allclose([r.step for r in ref.report.rows], [r.step for r in mine.report.rows],
                       rtol=1e-9)
    assert np.allclose(ref.p, mine.p.numpy(), rtol=1e-8, atol=1e-12)


def test_line_search_contract():
    a, b, p0 = _problem(4, 1)
    obj = TorchQuadratic(a, b)
    p = torch.as_tensor(p0)
    v, g = obj.value_and_grad(p)
    res = qn.backtracking_line_search(obj.value, p, -g, g, v, initial_step=1e-3)
    assert res.success and res.value <= v
    with pytest.raises(qn.LineSearchError):
        qn.backtracking_line_search(obj.value, p, g, g, v)


@pytest.mark.gpu
def test_lbfgs_on_gpu_fwi_objective():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from cases import small_case
    from paper_2008_11778_b200 import gradients
    case = small_case(8, True)
    g = case["gold"]
    obj = gradients.FwiObjective(case["grid"], list(g["obs"]), case["wavelet"],
                                 case["geometry"], case["config"])
    res = qn.minimize_lbfgs(obj, g["m"].ravel(), memory=3, max_iters=4)
    j = [r.objective for r in res.report.rows]
    assert j[-1] < j[0]
    res2 = qn.minimize_ncg(gradients.FwiObjective(case["grid"], list(g["obs"]), case["wavelet"],
                                                  case["geometry"], case["config"]),
                           g["m"].ravel(), max_iters=3)
    assert res2.report.rows[-1].objective < res2.report.rows[0].objective

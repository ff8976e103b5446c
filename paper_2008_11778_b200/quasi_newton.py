"""The paper's comparators on device vectors: limited-memory
BFGS and Polak-Ribiere+ nonlinear CG, plus the Armijo backtracking search they
use.  Same iterates, counters, report rows and fall-back rules as
seisopt/optim/quasi_newton.py:16-208 and seisopt/optim/linesearch.py:29-70;
the code is organised around direction-rule objects driven by one loop.

Iterates, gradients and curvature pairs stay torch tensors on the problem's
device; inner products and vector updates run in libseisgpu's fused vector
kernels (``devvec``), and only scalars (inner products, objective values)
reach the host.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from . import devvec
from .anderson import OptimizeResult, OptimizerReport, _budget_allows, default_eta

CURVATURE_SKIP_TOL = 1e-12  # seisopt/optim/quasi_newton.py:13


def _torch():
    import torch
    return torch


def _ip(a, b):
    return devvec.dot(a, b)


def _len(a):
    return devvec.norm(a)


def _lin(coefs, xs, y=None):
    """y + sum_i coefs[i] xs[i] as a new vector (one device pass)."""
    return devvec.axpy(coefs, xs, y)


class LineSearchError(Exception):
    """Ascent direction or non-positive initial step (seisopt/optim/linesearch.py:17)."""


@dataclass
class LineSearchResult:
    step: float
    value: float
    trials: int
    success: bool
    curvature_ok: bool | None = None


def backtracking_line_search(value_fn, p, direction, grad_p, value_p, initial_step=1.0,
                             c1=1e-4, c2=0.9, max_backtracks=10, shrink=0.5, grad_fn=None,
                             budget_ok=None):
    """Armijo search over s0, s0*shrink, ... (seisopt/optim/linesearch.py:29-70)."""
    slope = _ip(direction, grad_p)
    if slope >= 0.0:
        raise LineSearchError(f"not a descent direction: <d, grad> = {slope:.3g}")
    if initial_step <= 0.0:
        raise LineSearchError("initial step must be positive")
    s = float(initial_step)
    for n_try in range(1, max_backtracks + 1):
        if budget_ok is not None and not budget_ok():
            return LineSearchResult(0.0, value_p, n_try - 1, False)
        trial_point = _lin([s], [direction], p)
        f = value_fn(trial_point)
        if np.isfinite(f) and f <= value_p + c1 * s * slope:
            ok = None if grad_fn is None else bool(
                _ip(direction, grad_fn(trial_point)) >= c2 * slope)
            return LineSearchResult(s, float(f), n_try, True, ok)
        s *= shrink
    return LineSearchResult(0.0, value_p, max_backtracks, False)


class LBFGSHistory:
    """Curvature pairs (dp, dg, 1/<dp,dg>) of the last ``memory`` accepted
    steps (seisopt/optim/quasi_newton.py:16-54)."""

    def __init__(self, memory):
        self.memory = memory
        self._q = deque()

    @property
    def pairs(self):
        return list(self._q)

    def push(self, dp, dg):
        rho_inv = _ip(dp, dg)
        if rho_inv <= CURVATURE_SKIP_TOL * _len(dp) * _len(dg):
            return False
        self._q.append((dp, dg, 1.0 / rho_inv))
        while len(self._q) > self.memory:
            self._q.popleft()
        return True

    def clear(self):
        self._q.clear()

    def apply(self, v):
        """H_k v by the two-loop recursion, H_0 = <dp,dg>/<dg,dg> I."""
        q = v.clone()
        coeff = []
        for dp, dg, rho in reversed(self._q):
            a = rho * _ip(dp, q)
            devvec.axpy([-a], [dg], q, out=q)
            coeff.append(a)
        if self._q:
            dp, dg, _ = self._q[-1]
            devvec.scale(_ip(dp, dg) / _ip(dg, dg), q, out=q)
        for (dp, dg, rho), a in zip(self._q, reversed(coeff)):
            devvec.axpy([a - rho * _ip(dg, q)], [dp], q, out=q)
        return q


class _LBFGSRule:
    """Direction -H g; resets to steepest descent on a non-descent direction
    or a failed search (seisopt/optim/quasi_newton.py:139-152)."""

    method = "lbfgs"

    def __init__(self, memory):
        self.hist = LBFGSHistory(memory)

    def direction(self, g, eta0):
        d = devvec.scale(-1.0, self.hist.apply(g))
        if _ip(d, g) >= 0.0:
            self.hist.clear()
            d = devvec.scale(-1.0, g)
        return d, (1.0 if self.hist._q else eta0)

    def accepted(self, p, g, p_new, g_new, d, fell_back):
        if fell_back:
            self.hist.clear()
        self.hist.push(_lin([-1.0], [p], p_new), _lin([-1.0], [g], g_new))


class _PRPlusRule:
    """d = -g + max(0, PR) d_prev, restarting on non-descent; initial trial
    step twice the previous step length (seisopt/optim/quasi_newton.py:176-203)."""

    method = "ncg"

    def __init__(self):
        self.g_prev = self.d_prev = self.s_prev = None

    def direction(self, g, eta0):
        if self.g_prev is None:
            d = devvec.scale(-1.0, g)
        else:
            beta = max(0.0, _ip(g, _lin([-1.0], [self.g_prev], g)) /
                       _ip(self.g_prev, self.g_prev))
            d = _lin([-1.0, beta], [g, self.d_prev])
            if _ip(d, g) >= 0.0:
                d = devvec.scale(-1.0, g)
        self.d_prev = d
        return d, (eta0 if self.s_prev is None else 2.0 * self.s_prev)

    def accepted(self, p, g, p_new, g_new, d, fell_back):
        self.g_prev, self.d_prev = g, d
        dl = _len(d)
        self.s_prev = _len(_lin([-1.0], [p], p_new)) / dl if dl else None


def _drive(problem, p0, rule, budget, max_iters, grad_tol, c1, c2, max_backtracks, line_search):
    """One value_and_grad per iterate, carried across steps
    (seisopt/optim/quasi_newton.py:75-120)."""
    torch = _torch()
    host = not isinstance(p0, torch.Tensor)
    if host:
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
        p = torch.as_tensor(np.asarray(p0, dtype=np.float64).reshape(-1), device=dev)
    else:
        p = p0.reshape(-1).clone()
    report = OptimizerReport(method=rule.method)
    extras = {}

    def result(x):
        return OptimizeResult(p=x.double().cpu().numpy() if host else x, report=report,
                              extras=extras)

    def evaluate(x):
        v, g = problem.value_and_grad(x)
        if not isinstance(g, torch.Tensor):
            g = torch.as_tensor(g)
        return float(v), g.to(device=x.device, dtype=x.dtype).reshape(-1)

    if not _budget_allows(problem, budget, 1.0):
        return result(p)
    f, g = evaluate(p)
    eta0 = default_eta(p, g) if p.is_cuda else default_eta(p.cpu().numpy(), g.cpu().numpy())
    extras["eta"] = eta0
    k = 0
    while True:
        gnorm = _len(g)
        stop = (grad_tol and gnorm <= grad_tol) or (max_iters is not None and k >= max_iters) \
            or gnorm == 0.0
        step, p_new, d, fell_back = 0.0, p, None, False
        if not stop:
            d, s0 = rule.direction(g, eta0)
            if line_search is not None:
                step = float(line_search(problem, p, f, g, d))
            else:
                ls = backtracking_line_search(
                    problem.value, p, d, g, f, initial_step=s0, c1=c1, c2=c2,
                    max_backtracks=max_backtracks,
                    budget_ok=lambda: _budget_allows(problem, budget, 0.5))
                if ls.success:
                    step = ls.step
                else:  # small steepest-descent step (quasi_newton.py:63-72)
                    step, d, fell_back = eta0, devvec.scale(-1.0, g), True
            p_new = _lin([step], [d], p)
        report.append(iteration=k, objective=f, grad_norm=gnorm,
                      grad_evals=problem.counters.grad_evals,
                      obj_evals=problem.counters.obj_evals, step=step)
        if stop:
            break
        if not _budget_allows(problem, budget, 1.0):
            p = p_new
            break
        f_new, g_new = evaluate(p_new)
        rule.accepted(p, g, p_new, g_new, d, fell_back)
        p, f, g = p_new, f_new, g_new
        k += 1
    return result(p)


def minimize_lbfgs(problem, p0, memory, budget=None, max_iters=None, grad_tol=0.0, c1=1e-4,
                   c2=0.9, max_backtracks=10, line_search=None):
    """L-BFGS with Armijo backtracking (seisopt/optim/quasi_newton.py:123-161)."""
    rule = _LBFGSRule(memory)
    res = _drive(problem, p0, rule, budget, max_iters, grad_tol, c1, c2, max_backtracks,
                 line_search)
    res.extras["history"] = rule.hist
    return res


def minimize_ncg(problem, p0, budget=None, max_iters=None, grad_tol=0.0, c1=1e-4, c2=0.9,
                 max_backtracks=10, line_search=None):
    """Polak-Ribiere+ nonlinear CG (seisopt/optim/quasi_newton.py:164-208)."""
    return _drive(problem, p0, _PRPlusRule(), budget, max_iters, grad_tol, c1, c2,
                  max_backtracks, line_search)

"""L-BFGS and Polak-Ribiere+ nonlinear CG on device vectors -- the paper's
comparators, restating seisopt/optim/quasi_newton.py:16-208
and the Armijo backtracking of seisopt/optim/linesearch.py:29-70.

Iterates, gradients and update pairs stay in torch tensors on the problem's
device; only scalars (dots, norms, objective values) reach the host.  Works
with any objective following the protocol of seisopt/optim/problems.py:1-5
that accepts torch tensors (the objectives of ``gradients``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .anderson import OptimizeResult, OptimizerReport, _budget_allows, default_eta

CURVATURE_SKIP_TOL = 1e-12


def _torch():
    import torch
    return torch


def _dot(a, b):
    return float((a.double() * b.double()).sum().item())


def _norm(a):
    return float(a.double().norm().item())


class LineSearchError(Exception):
    """Precondition violation (seisopt/optim/linesearch.py:17-18)."""


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
    """Largest s in {s0, s0/2, ...} with J(p + s d) <= J(p) + c1 s <d, g>
    (seisopt/optim/linesearch.py:29-70)."""
    slope = _dot(direction, grad_p)
    if slope >= 0.0:
        raise LineSearchError(f"not a descent direction: <d, grad> = {slope:.3g}")
    if initial_step <= 0.0:
        raise LineSearchError("initial step must be positive")
    step = float(initial_step)
    for trial in range(1, max_backtracks + 1):
        if budget_ok is not None and not budget_ok():
            return LineSearchResult(0.0, value_p, trial - 1, False)
        cand = value_fn(p + step * direction)
        if np.isfinite(cand) and cand <= value_p + c1 * step * slope:
            curv = None
            if grad_fn is not None:
                curv = bool(_dot(direction, grad_fn(p + step * direction)) >= c2 * slope)
            return LineSearchResult(step, float(cand), trial, True, curv)
        step *= shrink
    return LineSearchResult(0.0, value_p, max_backtracks, False)


@dataclass
class LBFGSHistory:
    """Update pairs with positive curvature (seisopt/optim/quasi_newton.py:16-54)."""

    memory: int
    pairs: list = field(default_factory=list)

    def push(self, dp, dg):
        curv = _dot(dp, dg)
        if curv <= CURVATURE_SKIP_TOL * _norm(dp) * _norm(dg):
            return False
        self.pairs.append((dp, dg, 1.0 / curv))
        if len(self.pairs) > self.memory:
            self.pairs.pop(0)
        return True

    def clear(self):
        self.pairs.clear()

    def apply(self, vec):
        """Two-loop recursion with the <dp,dg>/<dg,dg> initial scaling."""
        q = vec.clone()
        alphas = []
        for dp, dg, rho in reversed(self.pairs):
            a = rho * _dot(dp, q)
            q -= a * dg
            alphas.append(a)
        if self.pairs:
            dp, dg, _ = self.pairs[-1]
            q *= _dot(dp, dg) / _dot(dg, dg)
        for (dp, dg, rho), a in zip(self.pairs, reversed(alphas)):
            q += (a - rho * _dot(dg, q)) * dp
        return q


def _as_vec(p0, like=None):
    torch = _torch()
    if isinstance(p0, torch.Tensor):
        return p0.reshape(-1).clone(), False
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")
    return torch.as_tensor(np.asarray(p0, dtype=np.float64).reshape(-1), device=dev), True


def _qn_loop(problem, p0, method, direction_fn, on_accept, budget, max_iters, grad_tol, c1, c2,
             max_backtracks, line_search):
    """Shared driver (seisopt/optim/quasi_newton.py:75-120)."""
    torch = _torch()
    p, numpy_out = _as_vec(p0)
    report = OptimizerReport(method=method)
    extras = {}

    def finish(p):
        return OptimizeResult(p=p.double().cpu().numpy() if numpy_out else p, report=report,
                              extras=extras)

    def vg(x):
        v, g = problem.value_and_grad(x)
        g = g if isinstance(g, torch.Tensor) else torch.as_tensor(g, device=x.device)
        return float(v), g.to(device=x.device, dtype=x.dtype).reshape(-1)

    if not _budget_allows(problem, budget, 1.0):
        return finish(p)
    value, grad = vg(p)
    eta0 = default_eta(p, grad) if p.is_cuda else default_eta(p.cpu().numpy(), grad.cpu().numpy())
    extras["eta"] = eta0
    k = 0
    while True:
        gn = _norm(grad)
        done = (grad_tol and gn <= grad_tol) or (max_iters is not None and k >= max_iters) \
            or gn == 0.0
        step, p_next, d, fell_back = 0.0, p, None, False
        if not done:
            d, initial = direction_fn(grad, eta0)
            if line_search is not None:
                step = float(line_search(problem, p, value, grad, d))
            else:
                res = backtracking_line_search(
                    problem.value, p, d, grad, value, initial_step=initial, c1=c1, c2=c2,
                    max_backtracks=max_backtracks,
                    budget_ok=lambda: _budget_allows(problem, budget, 0.5))
                if res.success:
                    step = res.step
                else:
                    step, d, fell_back = eta0, -grad, True
            p_next = p + step * d
        report.append(iteration=k, objective=value, grad_norm=gn,
                      grad_evals=problem.counters.grad_evals,
                      obj_evals=problem.counters.obj_evals, step=step)
        if done:
            break
        if not _budget_allows(problem, budget, 1.0):
            p = p_next
            break
        value_next, grad_next = vg(p_next)
        on_accept(p, grad, p_next, grad_next, d, fell_back)
        p, value, grad = p_next, value_next, grad_next
        k += 1
    return finish(p)


def minimize_lbfgs(problem, p0, memory, budget=None, max_iters=None, grad_tol=0.0, c1=1e-4,
                   c2=0.9, max_backtracks=10, line_search=None):
    """seisopt/optim/quasi_newton.py:123-161."""
    hist = LBFGSHistory(memory=memory)

    def direction(grad, eta0):
        d = -hist.apply(grad)
        if _dot(d, grad) >= 0.0:
            hist.clear()
            d = -grad
        return d, (1.0 if hist.pairs else eta0)

    def on_accept(p, grad, p_next, grad_next, d, fell_back):
        if fell_back:
            hist.clear()
        hist.push(p_next - p, grad_next - grad)

    res = _qn_loop(problem, p0, "lbfgs", direction, on_accept, budget, max_iters, grad_tol, c1,
                   c2, max_backtracks, line_search)
    res.extras["history"] = hist
    return res


def minimize_ncg(problem, p0, budget=None, max_iters=None, grad_tol=0.0, c1=1e-4, c2=0.9,
                 max_backtracks=10, line_search=None):
    """Polak-Ribiere+ (seisopt/optim/quasi_newton.py:164-208)."""
    st = {"g": None, "d": None, "s": None}

    def direction(grad, eta0):
        if st["g"] is None:
            d = -grad
        else:
            beta = max(0.0, _dot(grad, grad - st["g"]) / _dot(st["g"], st["g"]))
            d = -grad + beta * st["d"]
            if _dot(d, grad) >= 0.0:
                d = -grad
        st["d"] = d
        return d, (2.0 * st["s"] if st["s"] is not None else eta0)

    def on_accept(p, grad, p_next, grad_next, d, fell_back):
        st["g"], st["d"] = grad, d
        dn = _norm(d)
        st["s"] = _norm(p_next - p) / dn if dn else None

    return _qn_loop(problem, p0, "ncg", direction, on_accept, budget, max_iters, grad_tol, c1,
                    c2, max_backtracks, line_search)

"""Anderson acceleration on the device -- drop-in for seisopt.optim.anderson.

* ``AAWindow`` (seisopt/optim/anderson.py:55-112) is a libseisgpu window:
  ring buffers of residual / G differences in HBM plus an fp64 Gram matrix
  (see csrc/sg_aa.cu).  ``push`` accepts NumPy or torch CUDA vectors.
* ``aa_weights`` (:115-123), ``aa_step`` (:126-148) as in the reference.
* ``minimize_aa`` (:283-353) + ``_blend_search`` (:356-376) run with every
  N-vector resident on the GPU when the problem accepts torch tensors (the
  objectives in ``gradients``); only scalars cross to the host.  The report,
  counters, extras (eta, inequality_log, lambdas) and the budget veto match
  the reference.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import EmptyWindowError  # noqa: F401

RANK_TOL = 1e-12


def _torch():
    import torch
    return torch


def _dt(t):
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.SG_F32
    if t.dtype == torch.float64:
        return _lib.SG_F64
    raise ValueError("vectors must be float32 or float64")


def _stream(t):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def vec_stats(x):
    """{min, max, max_abs, norm, nonfinite} of a CUDA vector (one fused pass)."""
    out = (C.c_double * 5)()
    x = x.contiguous()
    _lib.check(_lib.load().sg_vec_stats(x.numel(), _dt(x), _lib.dptr(x), out, _stream(x)),
               "vec_stats")
    return dict(min=out[0], max=out[1], max_abs=out[2], norm=out[3], nonfinite=int(out[4]))


def vec_axpby(a, x, b, y, out=None):
    torch = _torch()
    out = torch.empty_like(x) if out is None else out
    _lib.check(_lib.load().sg_vec_axpby(x.numel(), _dt(x), float(a), _lib.dptr(x), float(b),
                                        _lib.dptr(y), _lib.dptr(out), _stream(x)), "axpby")
    return out


def vec_lerp(x, y, lam, out=None):
    torch = _torch()
    out = torch.empty_like(x) if out is None else out
    _lib.check(_lib.load().sg_vec_lerp(x.numel(), _dt(x), _lib.dptr(x), _lib.dptr(y),
                                       float(lam), _lib.dptr(out), _stream(x)), "lerp")
    return out


def blend_dots(g, p, pbar, ptil):
    out = (C.c_double * 2)()
    _lib.check(_lib.load().sg_vec_blend_dots(g.numel(), _dt(g), _lib.dptr(g), _lib.dptr(p),
                                             _lib.dptr(pbar), _lib.dptr(ptil), out, _stream(g)),
               "blend_dots")
    return out[0], out[1]


@dataclass
class WeightSolution:
    """seisopt/optim/anderson.py:25-38."""

    gamma: np.ndarray
    alpha: np.ndarray
    residual_norm: float


class AAWindow:
    """Sliding AA history held on the GPU (seisopt/optim/anderson.py:55-112)."""

    def __init__(self, dim, memory, dtype="float64", device=None, qr="auto", shard_group=None):
        """``shard_group``: a torch.distributed process group (or True for the
        default group) over which the N-vectors are sharded -- ``dim`` is then
        this rank's slice length and every inner product of the window is
        summed over the group (sg_aa_set_reducer)."""
        torch = _torch()
        if qr not in ("auto", "always"):
            raise ValueError("qr must be 'auto' (Gram, device QR when it cannot resolve "
                             "the window) or 'always'")
        if memory < 0:
            raise ValueError("memory must be non-negative")
        self.dim = int(dim)
        self.memory = int(memory)
        self.tdtype = torch.float32 if dtype in ("float32", torch.float32, np.float32) \
            else torch.float64
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self.lib.sg_aa_create(self.dim, self.memory,
                                         4 if self.tdtype == torch.float32 else 8,
                                         self.device.index, C.byref(h)), "sg_aa_create")
        self.h = h
        self._numpy_io = False
        if qr == "always":
            _lib.check(self.lib.sg_aa_set_qr(h, 1), "sg_aa_set_qr")
        self._reducer = None
        if shard_group is not None and shard_group is not False:
            self._install_reducer(None if shard_group is True else shard_group)

    def _install_reducer(self, group, force=False):
        """force: install the hook on a one-rank group too (tests of the
        collective path with one GPU)."""
        torch = _torch()
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            raise RuntimeError("a sharded AAWindow needs an initialised process group")
        if dist.get_world_size(group) == 1 and not force:
            return
        nccl = dist.get_backend(group) == "nccl"
        dev = self.device

        def reduce(buf, n, _ctx):
            try:
                host = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))
                if nccl:
                    t = host.to(dev)
                    dist.all_reduce(t, group=group)
                    host.copy_(t)
                else:
                    dist.all_reduce(host, group=group)
                return 0
            except Exception:  # surfaces as SG_ERR_STATE from the push
                return 1

        self._reducer = _lib.REDUCE_FN(reduce)  # keep the thunk alive
        _lib.check(self.lib.sg_aa_set_reducer(self.h, C.cast(self._reducer, C.c_void_p), None),
                   "sg_aa_set_reducer")

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.sg_aa_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _dev(self, x):
        torch = _torch()
        if isinstance(x, torch.Tensor):
            return x.to(device=self.device, dtype=self.tdtype).contiguous().reshape(-1)
        self._numpy_io = True
        return torch.as_tensor(np.asarray(x, dtype=np.float64).reshape(-1), device=self.device,
                               dtype=self.tdtype)

    def _set_stream(self):
        torch = _torch()
        self.lib.sg_aa_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(self.device)
                                                     .cuda_stream))

    @property
    def m_k(self):
        return int(self.lib.sg_aa_m_k(self.h))

    def clear(self):
        _lib.check(self.lib.sg_aa_clear(self.h), "clear")

    def push(self, p, g_value):
        """Record iterate p and its operator image G(p) (anderson.py:80-96)."""
        pd, gd = self._dev(p), self._dev(g_value)
        if pd.numel() != self.dim or gd.numel() != self.dim:
            raise ValueError(f"vectors must have {self.dim} entries")
        self._set_stream()
        _lib.check(self.lib.sg_aa_push(self.h, _lib.dptr(pd), _lib.dptr(gd)), "push")

    def qr_info(self):
        """(current window factored by the device QR?, QR passes run so far)."""
        act, passes = C.c_int32(), C.c_int64()
        _lib.check(self.lib.sg_aa_qr_info(self.h, C.byref(act), C.byref(passes)), "qr_info")
        return bool(act.value), int(passes.value)

    def f_k_norm(self):
        out = C.c_double()
        _lib.check(self.lib.sg_aa_fk_norm(self.h, C.byref(out)), "f_k_norm")
        return out.value


def aa_weights(window: AAWindow) -> WeightSolution:
    """seisopt/optim/anderson.py:115-123."""
    if window.m_k == 0:
        raise EmptyWindowError("aa_weights needs at least one stored difference")
    m = window.m_k
    gamma = np.zeros(m)
    alpha = np.zeros(m + 1)
    resid = C.c_double()
    mk = C.c_int32()
    _lib.check(window.lib.sg_aa_weights(window.h, _lib.hptr_d(gamma), _lib.hptr_d(alpha),
                                        C.byref(resid), C.byref(mk)), "aa_weights")
    return WeightSolution(gamma=gamma[: mk.value], alpha=alpha[: mk.value + 1],
                          residual_norm=resid.value)


def aa_step(window: AAWindow, beta=1.0, weights=None, out=None):
    """Next iterate (seisopt/optim/anderson.py:126-148).  Returns a torch CUDA
    tensor, or NumPy float64 when the window was fed NumPy vectors."""
    torch = _torch()
    res = torch.empty(window.dim, device=window.device, dtype=window.tdtype) if out is None \
        else out
    window._set_stream()
    if weights is not None and window.m_k > 0:
        gamma = np.ascontiguousarray(weights.gamma, dtype=np.float64)
        _lib.check(window.lib.sg_aa_step(window.h, float(beta), _lib.hptr_d(gamma), None,
                                         _lib.dptr(res)), "aa_step")
    else:
        _lib.check(window.lib.sg_aa_step(window.h, float(beta), None, None, _lib.dptr(res)),
                   "aa_step")
    if window._numpy_io and out is None:
        return res.double().cpu().numpy()
    return res


def picard_step(operator, p):
    """seisopt/optim/anderson.py:151-153."""
    return operator(p)


def default_eta(p0, g0):
    """seisopt/optim/problems.py:85-93 (device reductions for CUDA vectors)."""
    torch = _torch()
    if isinstance(g0, torch.Tensor) and g0.is_cuda:
        g_inf = vec_stats(g0)["max_abs"]
        sp = vec_stats(p0)
        scale = sp["max"] - sp["min"]
        pabs = sp["max_abs"]
    else:
        g_inf = float(np.max(np.abs(g0)))
        scale = float(np.ptp(p0))
        pabs = float(np.max(np.abs(p0)))
    if g_inf == 0.0:
        return 1.0
    if scale == 0.0:
        scale = max(1.0, pabs)
    return 0.01 * scale / g_inf


# ---------------------------------------------------------------------------
# report types (seisopt/optim/report.py)
# ---------------------------------------------------------------------------

_COLUMNS = ("iteration", "objective", "grad_norm", "grad_evals", "obj_evals", "step")


@dataclass
class IterationRecord:
    iteration: int
    objective: float
    grad_norm: float
    grad_evals: int
    obj_evals: int
    step: float


@dataclass
class OptimizerReport:
    method: str
    rows: list = field(default_factory=list)

    def append(self, **kw):
        self.rows.append(IterationRecord(**kw))

    @property
    def final_objective(self):
        return self.rows[-1].objective if self.rows else float("nan")

    def objectives(self):
        return np.array([r.objective for r in self.rows])

    def grad_norms(self):
        return np.array([r.grad_norm for r in self.rows])

    def to_csv(self, path):
        def fmt(v):
            return str(int(v)) if isinstance(v, (int, np.integer)) else f"{float(v):.17g}"
        lines = [",".join(_COLUMNS)]
        for r in self.rows:
            lines.append(",".join(fmt(v) for v in (r.iteration, r.objective, r.grad_norm,
                                                     r.grad_evals, r.obj_evals, r.step)))
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")


@dataclass
class OptimizeResult:
    p: object
    report: OptimizerReport
    extras: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# optimizer drivers
# ---------------------------------------------------------------------------


def _budget_allows(problem, budget, cost):
    """seisopt/optim/anderson.py:229-232."""
    if budget is None:
        return True
    return problem.counters.grad_equivalents + cost <= budget + 1e-9


def _on_device(problem, p0, device):
    """Device-resident loop when the problem takes torch tensors."""
    torch = _torch()
    if isinstance(p0, torch.Tensor) and p0.is_cuda:
        return True
    return device is not None or getattr(problem, "prop", None) is not None or \
        getattr(problem, "kernel", None) is not None


def minimize_aa(problem, p0, memory, eta=None, budget=None, max_iters=None, grad_tol=0.0,
                c1=1e-4, max_backtracks=10, *, dtype=None, device=None):
    """Anderson-accelerated steepest descent, Alg. 2 as implemented in
    seisopt/optim/anderson.py:283-353, with all N-vectors on the GPU.

    ``p0`` may be NumPy (the result's ``p`` is then NumPy float64) or a torch
    CUDA tensor.  The problem must accept torch CUDA vectors (the objectives of
    ``paper_2008_11778_b200.gradients`` do)."""
    torch = _torch()
    numpy_out = not isinstance(p0, torch.Tensor)
    if dtype is None:
        dtype = p0.dtype if isinstance(p0, torch.Tensor) else torch.float64
        prop = getattr(problem, "prop", None) or getattr(getattr(problem, "kernel", None),
                                                         "ws", None)
        if prop is not None and numpy_out:
            dtype = prop.tdtype
    dev = device
    if dev is None:
        dev = p0.device if isinstance(p0, torch.Tensor) else torch.device(
            "cuda", torch.cuda.current_device())
    p = torch.as_tensor(p0 if isinstance(p0, torch.Tensor) else np.asarray(p0, np.float64),
                        device=dev, dtype=dtype).reshape(-1).contiguous().clone()
    window = AAWindow(p.numel(), memory, dtype=p.dtype, device=p.device)
    report = OptimizerReport(method="aa")
    inequality_log, lambdas = [], []
    pbar = torch.empty_like(p)
    ptil = torch.empty_like(p)
    cand = torch.empty_like(p)
    k = 0
    while True:
        if not _budget_allows(problem, budget, 1.0):
            break
        value, grad = problem.value_and_grad(p)
        grad = grad if isinstance(grad, torch.Tensor) else torch.as_tensor(grad, device=p.device)
        grad = grad.to(p.dtype).reshape(-1).contiguous()
        if eta is None:
            eta = default_eta(p, grad)
        grad_norm = vec_stats(grad)["norm"]
        done = (grad_tol and grad_norm <= grad_tol) or (max_iters is not None and k >= max_iters)
        lam = 0.0
        p_next = None
        if not done:
            vec_axpby(1.0, p, -eta, grad, out=pbar)  # p_bar = p - eta grad
            window.push(p, pbar)
            if window.m_k == 0:
                p_next = pbar.clone()
            else:
                w = aa_weights(window)
                inequality_log.append((w.residual_norm, window.f_k_norm()))
                aa_step(window, weights=w, out=ptil)
                lam, p_next = _blend_search(problem, value, grad, p, pbar, ptil, c1,
                                            max_backtracks,
                                            lambda: _budget_allows(problem, budget, 0.5), cand)
                if lam == 0.0:
                    window.clear()
                    p_next = pbar.clone()
                else:
                    p_next = p_next.clone()
            lambdas.append(lam)
        report.append(iteration=k, objective=value, grad_norm=grad_norm,
                      grad_evals=problem.counters.grad_evals,
                      obj_evals=problem.counters.obj_evals, step=lam)
        if done:
            break
        p = p_next
        k += 1
    out_p = p.double().cpu().numpy() if numpy_out else p
    return OptimizeResult(p=out_p, report=report,
                          extras={"eta": eta, "inequality_log": inequality_log,
                                  "lambdas": lambdas})


def _blend_search(problem, value_k, grad_k, p_k, p_bar, p_tilde, c1, max_backtracks, budget_ok,
                  cand=None):
    """seisopt/optim/anderson.py:356-376 on device vectors."""
    base, cross = blend_dots(grad_k, p_k, p_bar, p_tilde)
    lam = 1.0
    for _ in range(max_backtracks):
        if not budget_ok():
            return 0.0, p_bar
        cand = vec_lerp(p_bar, p_tilde, lam, out=cand)
        slope = base + lam * cross
        bound = value_k + c1 * min(slope, 0.0)
        trial = problem.value(cand)
        if math.isfinite(trial) and trial <= bound:
            return lam, cand
        lam *= 0.5
    return 0.0, p_bar


def minimize_sd(problem, p0, eta=None, budget=None, max_iters=None, grad_tol=0.0,
                line_search=False, c1=1e-4, max_backtracks=10):
    """Steepest descent with a fixed step (default) or Armijo backtracking
    (seisopt/optim/anderson.py:235-280) on device vectors."""
    from .quasi_newton import backtracking_line_search
    torch = _torch()
    numpy_out = not isinstance(p0, torch.Tensor)
    prop = getattr(problem, "prop", None)
    dtype = p0.dtype if not numpy_out else (prop.tdtype if prop is not None else torch.float64)
    dev = p0.device if not numpy_out else torch.device("cuda", torch.cuda.current_device())
    p = torch.as_tensor(p0 if not numpy_out else np.asarray(p0, np.float64), device=dev,
                        dtype=dtype).reshape(-1).contiguous().clone()
    report = OptimizerReport(method="sd")
    k = 0
    while True:
        if not _budget_allows(problem, budget, 1.0):
            break
        value, grad = problem.value_and_grad(p)
        grad = grad if isinstance(grad, torch.Tensor) else torch.as_tensor(grad, device=p.device)
        grad = grad.to(p.dtype).reshape(-1).contiguous()
        if eta is None:
            eta = default_eta(p, grad)
        grad_norm = vec_stats(grad)["norm"]
        done = (grad_tol and grad_norm <= grad_tol) or (max_iters is not None and k >= max_iters)
        step = 0.0
        if not done:
            if line_search:
                res = backtracking_line_search(
                    problem.value, p, -grad, grad, value, initial_step=eta, c1=c1,
                    max_backtracks=max_backtracks,
                    budget_ok=lambda: _budget_allows(problem, budget, 0.5))
                step = res.step if res.success else eta * 0.5 ** max_backtracks
            else:
                step = eta
        report.append(iteration=k, objective=value, grad_norm=grad_norm,
                      grad_evals=problem.counters.grad_evals,
                      obj_evals=problem.counters.obj_evals, step=step)
        if done:
            break
        p = vec_axpby(1.0, p, -step, grad)
        k += 1
    return OptimizeResult(p=p.double().cpu().numpy() if numpy_out else p, report=report,
                          extras={"eta": eta})


# ---------------------------------------------------------------------------
# generic fixed-point acceleration (seisopt/optim/anderson.py:155-220)
# ---------------------------------------------------------------------------


@dataclass
class FixedPointTrace:
    """Iterates and residual diagnostics of a fixed-point run
    (seisopt/optim/anderson.py:155-165)."""

    iterates: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)
    combined_norms: list = field(default_factory=list)

    @property
    def final(self):
        return self.iterates[-1]


def aa_run(operator, p0, memory, iterations, beta=1.0, residual_tol=0.0, *, dtype=None,
           device=None):
    """Anderson acceleration of a fixed-point operator
    (seisopt/optim/anderson.py:168-203): per iteration push (p, G(p)), record
    ||f_k|| and the minimised combined residual, step with beta.

    The window lives on the GPU.  NumPy ``p0`` gives NumPy float64 iterates and
    the operator is called with NumPy vectors (like the reference); a torch
    CUDA ``p0`` keeps every iterate on the device and the operator receives
    torch tensors."""
    torch = _torch()
    numpy_io = not isinstance(p0, torch.Tensor)
    if dtype is None:
        dtype = torch.float64 if numpy_io else p0.dtype
    dev = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if numpy_io else p0.device)
    p = torch.as_tensor(np.asarray(p0, np.float64) if numpy_io else p0, device=dev,
                        dtype=dtype).reshape(-1).contiguous().clone()
    window = AAWindow(p.numel(), memory, dtype=p.dtype, device=p.device)

    def host(x):
        return x.double().cpu().numpy() if numpy_io else x

    trace = FixedPointTrace(iterates=[host(p.clone())])
    for _ in range(iterations):
        g_value = operator(host(p))
        g_dev = torch.as_tensor(g_value, device=p.device).to(p.dtype).reshape(-1).contiguous()
        window.push(p, g_dev)
        fk_norm = window.f_k_norm()
        if window.m_k == 0:
            p_next = aa_step(window, beta=beta)
            combined = fk_norm
        else:
            weights = aa_weights(window)
            p_next = aa_step(window, beta=beta, weights=weights)
            combined = weights.residual_norm
        trace.iterates.append(host(p_next))
        trace.residual_norms.append(fk_norm)
        trace.combined_norms.append(combined)
        p = p_next
        if residual_tol and fk_norm <= residual_tol:
            break
    return trace


def multisecant_oracle(p_mat, d_mat):
    """Minimiser S of ||S + I||_F subject to S D = P (closed form
    S = -I + (P + D)(D^T D)^{-1} D^T; seisopt/optim/anderson.py:206-222).  A
    dense n x n host helper for tests of the AA update, as in the reference."""
    p_mat = np.atleast_2d(np.asarray(p_mat, dtype=np.float64))
    d_mat = np.atleast_2d(np.asarray(d_mat, dtype=np.float64))
    if p_mat.shape != d_mat.shape:
        raise ValueError("P and D must have matching shapes")
    n, m = d_mat.shape
    if np.linalg.matrix_rank(d_mat) < m:
        raise np.linalg.LinAlgError("D is rank deficient; multi-secant oracle unavailable")
    coeff = np.linalg.solve(d_mat.T @ d_mat, d_mat.T)
    return -np.eye(n) + (p_mat + d_mat) @ coeff

"""FWI / LSRTM objectives and gradients on the B200 -- drop-in for
``seisopt.gradients`` (seisopt/gradients.py).

Same function names, argument meaning, return types, counters and error
behaviour as the reference; the arithmetic runs in libseisgpu.  Extra
keyword-only arguments select the device path: ``dtype`` ("float64" parity
mode, the default, or "float32" production mode), ``device``, and for the
objectives ``shard`` (multi-GPU shot ownership, see ``shards.py``).

NumPy inputs give NumPy float64 outputs (parity mode); torch CUDA inputs to
the objectives give torch outputs that never leave the device.
"""

from __future__ import annotations

import numpy as np

from .model import (EvalCounters, ObjectiveEval, ShotGather, SimConfig,  # noqa: F401
                    VelocityModel)
from .wavesim import Propagator, extend_to_pad, get_propagator, pad_spec  # noqa: F401


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# small host utilities with the reference's exact semantics
# ---------------------------------------------------------------------------


def pairwise_sum(arrays):
    """seisopt/gradients.py:40-50 (host utility; the GPU path reduces on device)."""
    items = [np.asarray(a) for a in arrays]
    if not items:
        raise ValueError("nothing to sum")
    while len(items) > 1:
        items = [items[i] + items[i + 1] if i + 1 < len(items) else items[i]
                 for i in range(0, len(items), 2)]
    return items[0]


def _check_matching(synthetic, observed):
    if len(synthetic) != len(observed):
        raise ValueError("gather counts differ")
    for s, o in zip(synthetic, observed):
        if s.samples.shape != o.samples.shape:
            raise ValueError(f"gather shapes differ: {s.samples.shape} vs {o.samples.shape}")


def trapezoid_weights(nt):
    """seisopt/gradients.py:63-67."""
    w = np.ones(nt)
    w[0] = 0.5
    w[-1] = 0.5
    return w


def misfit_l2(synthetic, observed):
    """Host misfit of gather lists (seisopt/gradients.py:70-79).  The device
    objectives fuse this reduction into the forward sweep."""
    _check_matching(synthetic, observed)
    total = 0.0
    for s, o in zip(synthetic, observed):
        d = s.samples - o.samples
        total += 0.5 * s.dt * float(np.einsum("t,tr->", trapezoid_weights(s.nt), d * d))
    return total


def adjoint_source(synthetic, observed):
    """seisopt/gradients.py:82-88."""
    _check_matching(synthetic, observed)
    return [ShotGather(source_index=s.source_index, samples=s.samples - o.samples, dt=s.dt)
            for s, o in zip(synthetic, observed)]


def data_norm(gathers):
    """seisopt/gradients.py:249-250."""
    return float(np.sqrt(sum(np.sum(g.samples * g.samples) for g in gathers)))


def laplacian_filter(image):
    """seisopt/gradients.py:280-292 (post-processing, host)."""
    arr = np.asarray(image, dtype=np.float64)
    p = np.pad(arr, 1, mode="edge")
    return -(p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:] - 4.0 * arr)


def _stack(gathers):
    if hasattr(gathers, "shape"):
        return gathers
    return np.stack([np.asarray(g.samples if hasattr(g, "samples") else g) for g in gathers])


def _gathers(arr, dt, start=0):
    a = arr.double().cpu().numpy() if hasattr(arr, "cpu") else np.asarray(arr)
    return [ShotGather(source_index=start + s, samples=a[s], dt=dt) for s in range(a.shape[0])]


# ---------------------------------------------------------------------------
# module functions (seisopt/gradients.py:98-277)
# ---------------------------------------------------------------------------


def fwi_synthetic(model, wavelet, geometry, config=SimConfig(), threads=1, workspace=None, *,
                  dtype="float64", device=None):
    """All-shot forward modelling (seisopt/gradients.py:98-115).  ``threads``
    is accepted for signature compatibility; all shots run batched on the GPU."""
    prop = workspace if isinstance(workspace, Propagator) else get_propagator(
        model.grid, geometry, wavelet, config, dtype, device)
    with prop._lock:  # set_model + sweep on a handle other threads may share
        prop.set_model(model.m)
        return _gathers(prop.synthetic(), geometry.dt)


def fwi_gradient(model, observed, wavelet, geometry, config=SimConfig(), counters=None,
                 threads=1, *, dtype="float64", device=None):
    """Misfit and exact gradient (seisopt/gradients.py:118-155)."""
    if len(observed) != geometry.n_sources:
        raise ValueError("observed data does not cover all sources")
    prop = get_propagator(model.grid, geometry, wavelet, config, dtype, device)
    with prop._lock:
        prop.set_model(model.m)
        value, grad = prop.gradient(_stack(observed))
        grad = grad.double().cpu().numpy()
    if counters is not None:
        counters.grad_evals += 1
    return ObjectiveEval(value=float(value), gradient=grad, gradient_eval_count_delta=1)


class BornKernel:
    """Born modelling about a fixed background (seisopt/gradients.py:158-220).

    ``cache`` ("auto" | True | False): keep every shot's background
    acceleration history in HBM (the reference always does, :177-184), or
    recompute it per apply (lock-step forward, checkpointed adjoint).
    """

    def __init__(self, background, wavelet, geometry, config=SimConfig(), threads=1, *,
                 dtype="float64", device=None, cache="auto", recon="auto", shard=None):
        self.background = background
        self.geometry = geometry
        self.threads = threads
        self.ws = Propagator(background.grid, geometry, wavelet, config, dtype=dtype,
                             device=device, recon=recon)
        self.ws.set_model(background.m)
        self.shard = shard
        self.born_applies = 0
        self.adjoint_applies = 0
        s0, cnt = self._range()
        self.cached = 0  # shots with a cached background history
        if cache is True or cache == "auto":
            # caches as many shots as fit in HBM; the rest are recomputed
            self.ws.born_cache((s0, cnt))
            self.cached = self.ws.born_cached()[1]
            if cache is True and self.cached < cnt:
                raise MemoryError(f"only {self.cached} of {cnt} background histories fit")

    def _range(self):
        if self.shard is None:
            return 0, self.geometry.n_sources
        return self.shard.shot0, self.shard.count

    @property
    def grid(self):
        return self.background.grid

    @property
    def grad_equivalents(self):
        """seisopt/gradients.py:186-189."""
        return 0.5 * (self.born_applies + self.adjoint_applies)

    def forward_device(self, m_r):
        out = self.ws.born_forward(m_r, self._range())
        self.born_applies += 1
        return out

    def adjoint_device(self, data, out=None):
        img = self.ws.born_adjoint(data, self._range(), out=out)
        if self.shard is not None:
            self.shard.allreduce_(img)
        self.adjoint_applies += 1
        return img

    def forward(self, m_r):
        """L m_r as ShotGathers (seisopt/gradients.py:191-205)."""
        d = self.forward_device(np.asarray(m_r, dtype=np.float64)
                                if not hasattr(m_r, "is_cuda") else m_r)
        return _gathers(d, self.geometry.dt, self._range()[0])

    def adjoint(self, data):
        """L^T y (seisopt/gradients.py:207-220)."""
        if not hasattr(data, "shape") and len(data) != self.geometry.n_sources:
            raise ValueError("data does not cover all sources")
        arr = _stack(data)
        s0, cnt = self._range()
        if arr.shape[0] == self.geometry.n_sources and cnt != arr.shape[0]:
            arr = arr[s0:s0 + cnt]
        return self.adjoint_device(arr).double().cpu().numpy()


def apply_born(background, reflectivity, wavelet, geometry, config=SimConfig(), kernel=None):
    """seisopt/gradients.py:223-233."""
    kernel = kernel or BornKernel(background, wavelet, geometry, config)
    return kernel.forward(reflectivity.m_r)


def apply_born_adjoint(background, data, wavelet, geometry, config=SimConfig(), kernel=None):
    """seisopt/gradients.py:236-246."""
    kernel = kernel or BornKernel(background, wavelet, geometry, config)
    return kernel.adjoint(data)


def lsrtm_objective(background, m_r, d_r, wavelet=None, geometry=None, config=SimConfig(),
                    kernel=None, counters=None):
    """J = 1/2 ||L m_r - d_r||^2, grad = L^T (L m_r - d_r) (seisopt/gradients.py:253-277)."""
    if kernel is None:
        if wavelet is None or geometry is None:
            raise ValueError("need wavelet and geometry when no kernel is given")
        kernel = BornKernel(background, wavelet, geometry, config)
    s0, cnt = kernel._range()
    dr = _stack(d_r)
    if dr.shape[0] != cnt:
        dr = dr[s0:s0 + cnt]
    value, grad = kernel.ws.lsrtm_gradient(np.asarray(m_r, dtype=np.float64)
                                           if not hasattr(m_r, "is_cuda") else m_r, dr, (s0, cnt))
    if kernel.shard is not None:
        value = kernel.shard.allreduce_value_grad(value, grad)
    kernel.born_applies += 1
    kernel.adjoint_applies += 1
    if counters is not None:
        counters.grad_evals += 1
    return ObjectiveEval(value=float(value), gradient=grad.double().cpu().numpy(),
                         gradient_eval_count_delta=1)


# ---------------------------------------------------------------------------
# objective protocol (seisopt/optim/problems.py:1-5; gradients.py:300-378)
# ---------------------------------------------------------------------------


class FwiObjective:
    """FWI misfit over squared slowness (seisopt/gradients.py:300-336).

    ``value(p)`` / ``value_and_grad(p)`` accept a NumPy vector (returns NumPy
    float64, the reference contract) or a torch CUDA tensor (returns a torch
    tensor on the device: the device-resident optimizer path).  The observed
    data are uploaded once.  With ``shard`` (shards.ShotShard) each rank runs
    its own shots and the misfit + gradient are all-reduced.
    """

    def __init__(self, grid, observed, wavelet, geometry, config=SimConfig(), threads=1, *,
                 dtype="float64", device=None, shard=None, recon="auto", batch=0,
                 checkpoint_every=0, mem_budget_bytes=0.0, chains=0):
        self.grid = grid
        self.wavelet = wavelet
        self.geometry = geometry
        self.config = config
        self.threads = threads
        self.counters = EvalCounters()
        self.shard = shard
        self.prop = Propagator(grid, geometry, wavelet, config, dtype=dtype, device=device,
                               recon=recon, batch=batch, checkpoint_every=checkpoint_every,
                               mem_budget_bytes=mem_budget_bytes, chains=chains)
        s0, cnt = self._range()
        obs = _stack(observed)
        if obs.shape[0] != geometry.n_sources:
            raise ValueError("observed data does not cover all sources")
        self.observed = observed
        self.obs_dev = self.prop.to_dev(obs[s0:s0 + cnt])

    def _range(self):
        if self.shard is None:
            return 0, self.geometry.n_sources
        return self.shard.shot0, self.shard.count

    def _valid(self, p):
        """Reference model check (seisopt/gradients.py:312-316), on device."""
        from .anderson import vec_stats
        torch = _torch()
        if isinstance(p, torch.Tensor) and p.is_cuda:
            st = vec_stats(p)
            return st["nonfinite"] == 0 and st["min"] > 0
        arr = np.asarray(p, dtype=np.float64)
        return bool(np.all(np.isfinite(arr)) and not np.any(arr <= 0))

    def value(self, p):
        if not self._valid(p):
            return float("inf")
        self.counters.obj_evals += 1
        self.prop.set_model(p)
        val = self.prop.misfit(self.obs_dev, self._range())
        if self.shard is not None:
            val = self.shard.allreduce_value(val)
        return float(val)

    def value_and_grad(self, p):
        from ._lib import ModelError
        torch = _torch()
        try:
            self.prop.set_model(p)
        except ModelError as exc:
            raise ValueError("model is not positive and finite") from exc
        val, grad = self.prop.gradient(self.obs_dev, self._range())
        if self.shard is not None:
            val = self.shard.allreduce_value_grad(val, grad)
        self.counters.grad_evals += 1
        if isinstance(p, torch.Tensor) and p.is_cuda:
            return float(val), grad.reshape(-1).to(p.dtype)
        return float(val), grad.double().cpu().numpy().ravel()


class LsrtmObjective:
    """Linearised least-squares migration objective (seisopt/gradients.py:339-378)."""

    def __init__(self, kernel: BornKernel, d_r):
        self.kernel = kernel
        self.d_r = d_r
        self.counters = EvalCounters()
        s0, cnt = kernel._range()
        dr = _stack(d_r)
        self.dr_dev = kernel.ws.to_dev(dr[s0:s0 + cnt] if dr.shape[0] != cnt else dr)

    @property
    def grid(self):
        return self.kernel.grid

    def _half_sq(self, p):
        """1/2 ||L m_r - d_r||^2 of this rank's shots (fused Born forward +
        fp64 residual reduction, sg_lsrtm_misfit), summed over ranks."""
        torch = _torch()
        k = self.kernel
        mr = p if isinstance(p, torch.Tensor) else np.asarray(p, dtype=np.float64)
        v = k.ws.lsrtm_misfit(mr, self.dr_dev, k._range())
        k.born_applies += 1
        if k.shard is not None:
            v = k.shard.allreduce_value(v)
        return v

    def residual_norm(self, p):
        """||L m_r - d_r||; one Born apply (seisopt/gradients.py:351-361)."""
        return float(np.sqrt(2.0 * self._half_sq(p)))

    def value(self, p):
        """seisopt/gradients.py:363-369."""
        self.counters.obj_evals += 1
        return float(self._half_sq(p))

    def value_and_grad(self, p):
        torch = _torch()
        k = self.kernel
        s0, cnt = k._range()
        mr = p if isinstance(p, torch.Tensor) else np.asarray(p, dtype=np.float64)
        val, grad = k.ws.lsrtm_gradient(mr, self.dr_dev, (s0, cnt))
        if k.shard is not None:
            val = k.shard.allreduce_value_grad(val, grad)
        k.born_applies += 1
        k.adjoint_applies += 1
        self.counters.grad_evals += 1
        if isinstance(p, torch.Tensor) and p.is_cuda:
            return float(val), grad.reshape(-1).to(p.dtype)
        return float(val), grad.double().cpu().numpy().ravel()

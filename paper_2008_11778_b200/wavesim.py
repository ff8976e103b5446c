"""Device propagator context and the reference's wavesim helpers.

``Propagator`` owns one libseisgpu handle: the B200 counterpart of
``seisopt.wavesim.Workspace`` (seisopt/wavesim.py:183-214) plus the
shot-batched sweep buffers, CUDA graphs of the time loops and the
reconstruction store.  Unlike the reference, which rebuilds a Workspace on
every ``fwi_gradient`` call (seisopt/gradients.py:136), a Propagator is built
once per (grid, geometry, wavelet, config, dtype) and only its model changes.

Host-side set-up that the reference does in NumPy (pad widths, sponge profiles,
bilinear taps) is restated here bit-identically, because the taps and sponge
values are part of the numerical contract (SURVEY s8b "stencil taps come from
the host").
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import threading
import warnings
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import ShotGather, SimConfig, StabilityError  # noqa: F401

# 8th-order stencil constants (BASELINE configs)
LAP8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)
CFL8_FACTOR = math.sqrt(4.0 / (205.0 / 72.0 + 2.0 * (8.0 / 5.0 + 1.0 / 5.0 + 8.0 / 315.0
                                                       + 1.0 / 560.0)))


@dataclass(frozen=True)
class PadSpec:
    """Per-side border widths (seisopt/wavesim.py:108-118)."""

    top: int
    bottom: int
    left: int
    right: int

    def padded_shape(self, grid):
        return (grid.nz + self.top + self.bottom, grid.nx + self.left + self.right)


def pad_spec(config) -> PadSpec:
    """seisopt/wavesim.py:121-123."""
    w = config.border_width
    return PadSpec(top=w if config.damp_top else 0, bottom=w, left=w, right=w)


def extend_to_pad(values, pad: PadSpec):
    """Edge replication onto the padded grid (seisopt/wavesim.py:126-128)."""
    return np.pad(values, ((pad.top, pad.bottom), (pad.left, pad.right)), mode="edge")


def restrict_to_interior(padded, pad: PadSpec, grid):
    """seisopt/wavesim.py:131-132."""
    return padded[pad.top: pad.top + grid.nz, pad.left: pad.left + grid.nx]


def sponge_profiles(grid, config):
    """1-D sponge factors (pz, px) whose outer product is the damping mask
    (seisopt/wavesim.py:150-165)."""
    pad = pad_spec(config)
    nzp, nxp = pad.padded_shape(grid)

    def prof(n, before, after):
        out = np.ones(n)
        kb = np.arange(before, 0, -1, dtype=np.float64)
        out[:before] = np.exp(-config.damping_strength * kb * kb)
        ka = np.arange(1, after + 1, dtype=np.float64)
        out[n - after:] = np.exp(-config.damping_strength * ka * ka)
        return out

    return prof(nzp, pad.top, pad.bottom), prof(nxp, pad.left, pad.right)


def damping_mask(grid, config):
    pz, px = sponge_profiles(grid, config)
    return np.outer(pz, px)


def bilinear_taps(points, grid, pad: PadSpec, shape):
    """Rows, cols, weights (4, n) -- seisopt/wavesim.py:168-180, same float ops."""
    nzp, nxp = shape
    xs = np.array([p[0] for p in points]) / grid.dx + pad.left
    zs = np.array([p[1] for p in points]) / grid.dz + pad.top
    i0 = np.minimum(np.floor(zs).astype(int), nzp - 2)
    j0 = np.minimum(np.floor(xs).astype(int), nxp - 2)
    tz = zs - i0
    tx = xs - j0
    rows = np.stack([i0, i0 + 1, i0, i0 + 1])
    cols = np.stack([j0, j0, j0 + 1, j0 + 1])
    w = np.stack([(1 - tz) * (1 - tx), tz * (1 - tx), (1 - tz) * tx, tz * tx])
    return rows, cols, w


def cfl_check(model, dt=None, cfl_safety=1.0, order=2):
    """Largest stable dt (seisopt/wavesim.py:92-100); the 8th-order stencil's
    bound is sqrt(4/6.5016) of the 5-point one."""
    grid = model.grid
    h = min(grid.dx, grid.dz)
    bound = cfl_safety * h / (model.c_max * math.sqrt(2.0))
    return bound * CFL8_FACTOR if order == 8 else bound


def _torch():
    import torch
    return torch


_RECON = {"full": _lib.SG_RECON_FULL, "checkpoint": _lib.SG_RECON_CHECKPOINT,
          "auto": _lib.SG_RECON_AUTO, "boundary": _lib.SG_RECON_BOUNDARY}


def torch_dtype(dtype):
    torch = _torch()
    if dtype in ("float32", "f32", np.float32, torch.float32):
        return torch.float32
    if dtype in ("float64", "f64", np.float64, torch.float64, None):
        return torch.float64
    raise ValueError(f"unsupported dtype {dtype!r}")


class Propagator:
    """One libseisgpu context: padded model, sponge, taps, wavelet, sweep buffers."""

    def __init__(self, grid, geometry, wavelet, config=SimConfig(), dtype="float64",
                 device=None, recon="auto", batch=0, checkpoint_every=0, use_graphs=True,
                 mem_budget_bytes=0.0, group=0, step_mode=0, chains=0, resident=0):
        torch = _torch()
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("libseisgpu needs a CUDA device; there is no CPU fallback")
        samples = np.asarray(getattr(wavelet, "samples", wavelet), dtype=np.float64)
        if samples.shape != (geometry.nt,):
            raise ValueError("wavelet length does not match geometry nt")
        geometry.validate_against(grid)
        self.grid, self.geometry, self.config = grid, geometry, config
        self.order = int(getattr(config, "order", 2))
        self.tdtype = torch_dtype(dtype)
        self.esz = 4 if self.tdtype == torch.float32 else 8
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.pad = pad_spec(config)
        self.shape = self.pad.padded_shape(grid)
        self.nt, self.n_shots, self.n_rec = geometry.nt, geometry.n_sources, geometry.n_receivers
        d = _lib.SgDesc()
        d.nz, d.nx = grid.nz, grid.nx
        d.pad_top, d.pad_bottom = self.pad.top, self.pad.bottom
        d.pad_left, d.pad_right = self.pad.left, self.pad.right
        d.nt, d.n_shots, d.n_rec = self.nt, self.n_shots, self.n_rec
        d.dtype, d.order = self.esz, self.order
        d.recon = _RECON[recon] if isinstance(recon, str) else int(recon)
        d.batch, d.checkpoint_every = int(batch), int(checkpoint_every)
        d.device = self.device.index
        d.use_graphs = 1 if use_graphs else 0
        d.group = int(group)
        d.step_mode = int(step_mode)
        d.chains = int(chains)
        d.resident = int(resident)
        d.dx, d.dz, d.dt = grid.dx, grid.dz, geometry.dt
        d.cfl_safety = config.cfl_safety
        d.mem_budget_bytes = float(mem_budget_bytes)
        self.desc = d
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.sg_create(C.byref(d), C.byref(h)), "sg_create")
        self.h = h
        pz, px = sponge_profiles(grid, config)
        _lib.check(self.lib.sg_set_sponge(h, _lib.hptr_d(pz), _lib.hptr_d(px)), "sponge")
        rr, rc, rw = bilinear_taps(geometry.receivers, grid, self.pad, self.shape)
        sr, sc, sw = bilinear_taps(geometry.sources, grid, self.pad, self.shape)
        self.rec_taps = (rr, rc, rw)
        self.src_taps = (sr, sc, sw)
        arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in (sr, sc)] + [
            np.ascontiguousarray(sw, dtype=np.float64)] + [
            np.ascontiguousarray(a, dtype=np.int32) for a in (rr, rc)] + [
            np.ascontiguousarray(rw, dtype=np.float64)]
        src_scale = 1.0 / (grid.dx * grid.dz)  # seisopt/wavesim.py:214
        _lib.check(self.lib.sg_set_geometry(
            h, _lib.hptr_i(arrs[0]), _lib.hptr_i(arrs[1]), _lib.hptr_d(arrs[2]),
            _lib.hptr_i(arrs[3]), _lib.hptr_i(arrs[4]), _lib.hptr_d(arrs[5]), src_scale),
            "geometry")
        self.wavelet = np.ascontiguousarray(samples)
        _lib.check(self.lib.sg_set_wavelet(h, _lib.hptr_d(self.wavelet)), "wavelet")
        # serialises set_model + sweep pairs of callers sharing this handle
        # (the module functions' cached propagators; ctypes releases the GIL)
        self._lock = threading.RLock()
        self.model_token = None

    # -- plumbing -----------------------------------------------------------
    def _stream(self):
        torch = _torch()
        s = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.sg_set_stream(self.h, C.c_void_p(s))

    def to_dev(self, x, dtype=None):
        torch = _torch()
        dt = self.tdtype if dtype is None else dtype
        if isinstance(x, torch.Tensor):
            return x.to(device=self.device, dtype=dt).contiguous()
        return torch.as_tensor(np.ascontiguousarray(x), device=self.device, dtype=dt)

    def _guard(self, what, value=None):
        """NaN/Inf guard: warn when the sweep diverged.  The
        reference returns the NaNs silently; so does this (same values), but
        says so."""
        n = C.c_int64()
        _lib.check(self.lib.sg_last_nonfinite(self.h, C.byref(n)), "last_nonfinite")
        self.last_nonfinite = n.value
        bad_val = value is not None and not np.isfinite(value)
        if n.value or bad_val:
            warnings.warn(f"{what}: non-finite result ({n.value} gradient entries"
                          f"{', misfit ' + repr(value) if bad_val else ''}): the sweep diverged",
                          RuntimeWarning, stacklevel=3)

    def close(self):
        if getattr(self, "h", None):
            self.lib.sg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _range(self, shots):
        if shots is None:
            return 0, self.n_shots
        s0, cnt = int(shots[0]), int(shots[1])
        return s0, cnt

    # -- model ----------------------------------------------------------------
    def set_model(self, m):
        """Squared slowness (nz, nx): numpy or torch.  Raises ModelError /
        StabilityError like the reference (seisopt/gradients.py:312-331,
        seisopt/wavesim.py:187-193)."""
        torch = _torch()
        t = m if isinstance(m, torch.Tensor) else torch.as_tensor(
            np.asarray(m, dtype=np.float64))
        t = t.reshape(self.grid.nz, self.grid.nx)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        t = t.to(self.device).contiguous()
        mdt = 4 if t.dtype == torch.float32 else 8
        self._stream()
        _lib.check(self.lib.sg_set_model(self.h, _lib.dptr(t), mdt), "set_model")
        self.model_token = object()

    # -- sweeps ---------------------------------------------------------------
    def synthetic(self, shots=None):
        torch = _torch()
        s0, cnt = self._range(shots)
        out = torch.empty((cnt, self.nt, self.n_rec), device=self.device, dtype=self.tdtype)
        self._stream()
        _lib.check(self.lib.sg_fwi_synthetic(self.h, s0, cnt, _lib.dptr(out)), "synthetic")
        return out

    def misfit(self, observed, shots=None):
        s0, cnt = self._range(shots)
        obs = self.to_dev(observed)
        v = C.c_double()
        self._stream()
        _lib.check(self.lib.sg_fwi_misfit(self.h, s0, cnt, _lib.dptr(obs), C.byref(v)), "misfit")
        return v.value

    def gradient(self, observed, shots=None, out=None, accumulate=False):
        torch = _torch()
        s0, cnt = self._range(shots)
        obs = self.to_dev(observed)
        if out is None:
            out = torch.empty((self.grid.nz, self.grid.nx), device=self.device, dtype=self.tdtype)
        v = C.c_double()
        self._stream()
        _lib.check(self.lib.sg_fwi_gradient(self.h, s0, cnt, _lib.dptr(obs), C.byref(v),
                                            _lib.dptr(out), 1 if accumulate else 0), "gradient")
        self._guard("fwi_gradient", v.value)
        return v.value, out

    def born_cache(self, shots=None, enable=True):
        s0, cnt = self._range(shots)
        self._stream()
        _lib.check(self.lib.sg_born_cache(self.h, s0, cnt, 1 if enable else 0), "born_cache")

    def born_cached(self):
        """(first shot, number of shots) whose background history is in HBM."""
        s0, cnt = C.c_int32(), C.c_int32()
        _lib.check(self.lib.sg_born_cached(self.h, C.byref(s0), C.byref(cnt)), "born_cached")
        return s0.value, cnt.value

    def born_forward(self, m_r, shots=None):
        torch = _torch()
        s0, cnt = self._range(shots)
        mr = self.to_dev(m_r).reshape(self.grid.nz, self.grid.nx).contiguous()
        out = torch.empty((cnt, self.nt, self.n_rec), device=self.device, dtype=self.tdtype)
        self._stream()
        _lib.check(self.lib.sg_born_forward(self.h, s0, cnt, _lib.dptr(mr), _lib.dptr(out)),
                   "born_forward")
        return out

    def born_adjoint(self, data, shots=None, out=None, accumulate=False):
        torch = _torch()
        s0, cnt = self._range(shots)
        dd = self.to_dev(data)
        if out is None:
            out = torch.empty((self.grid.nz, self.grid.nx), device=self.device, dtype=self.tdtype)
        self._stream()
        _lib.check(self.lib.sg_born_adjoint(self.h, s0, cnt, _lib.dptr(dd), _lib.dptr(out),
                                            1 if accumulate else 0), "born_adjoint")
        self._guard("born_adjoint")
        return out

    def lsrtm_gradient(self, m_r, d_r, shots=None, out=None, accumulate=False):
        torch = _torch()
        s0, cnt = self._range(shots)
        mr = self.to_dev(m_r).reshape(self.grid.nz, self.grid.nx).contiguous()
        dr = self.to_dev(d_r)
        if out is None:
            out = torch.empty((self.grid.nz, self.grid.nx), device=self.device, dtype=self.tdtype)
        v = C.c_double()
        self._stream()
        _lib.check(self.lib.sg_lsrtm_gradient(self.h, s0, cnt, _lib.dptr(mr), _lib.dptr(dr),
                                              C.byref(v), _lib.dptr(out),
                                              1 if accumulate else 0), "lsrtm_gradient")
        self._guard("lsrtm_gradient", v.value)
        return v.value, out

    def lsrtm_misfit(self, m_r, d_r, shots=None):
        """1/2 ||L m_r - d_r||^2 over the shots, reduced on the device."""
        s0, cnt = self._range(shots)
        mr = self.to_dev(m_r).reshape(self.grid.nz, self.grid.nx).contiguous()
        dr = self.to_dev(d_r)
        v = C.c_double()
        self._stream()
        _lib.check(self.lib.sg_lsrtm_misfit(self.h, s0, cnt, _lib.dptr(mr), _lib.dptr(dr),
                                            C.byref(v)), "lsrtm_misfit")
        return v.value

    def forward_history(self, shot):
        torch = _torch()
        g = torch.empty((self.nt, self.n_rec), device=self.device, dtype=self.tdtype)
        a = torch.empty((self.nt, *self.shape), device=self.device, dtype=self.tdtype)
        self._stream()
        _lib.check(self.lib.sg_forward_history(self.h, int(shot), _lib.dptr(g), _lib.dptr(a)),
                   "forward_history")
        return g, a

    def adjoint_history(self, ybar):
        torch = _torch()
        y = self.to_dev(ybar).reshape(self.nt, self.n_rec).contiguous()
        v = torch.empty((self.nt, *self.shape), device=self.device, dtype=self.tdtype)
        self._stream()
        _lib.check(self.lib.sg_adjoint_history(self.h, _lib.dptr(y), _lib.dptr(v)),
                   "adjoint_history")
        return v

    def query(self):
        b, r, by = C.c_int32(), C.c_int32(), C.c_double()
        _lib.check(self.lib.sg_query(self.h, C.byref(b), C.byref(r), C.byref(by)), "query")
        return dict(batch=b.value, recon={0: "full", 1: "checkpoint", 3: "boundary"}.get(r.value, r.value),
                    device_bytes=by.value)

    def resident_plan(self):
        """Cluster-resident sweep plan: whether the whole-sweep kernels run
        (fp32 grids whose shot fits one cluster's shared memory) and their
        launch shape."""
        out = (C.c_int32 * 6)()
        _lib.check(self.lib.sg_resident_plan(self.h, out), "resident_plan")
        return dict(on=bool(out[0]), cluster=out[1], cols_per_cta=out[2], threads=out[3],
                    clusters_resident=out[4], smem_bytes=out[5])

    def chains(self, count=None):
        """Concurrent shot chains a sweep over `count` shots runs as."""
        return int(self.lib.sg_chains(self.h, int(self.n_shots if count is None else count)))

    def phase_times(self):
        """Device ms of the last gradient's phases: forward sweep, residual +
        injection, adjoint sweep (with imaging), image reduction."""
        out = (C.c_float * 4)()
        _lib.check(self.lib.sg_phase_times(self.h, out), "phase_times")
        return dict(forward=out[0], residual=out[1], adjoint=out[2], reduce=out[3])

    def time_step_kernel(self, which, count=None, reps=50):
        ms = C.c_float()
        cnt = self.n_shots if count is None else count
        self._stream()
        _lib.check(self.lib.sg_time_step_kernel(self.h, int(which), int(cnt), int(reps),
                                                C.byref(ms)), "time_step_kernel")
        return ms.value


# ---------------------------------------------------------------------------
# propagator cache (the reference rebuilds its Workspace per call; we keep the
# device context, buffers and captured graphs alive across calls)
# ---------------------------------------------------------------------------

_CACHE: "OrderedDict[tuple, Propagator]" = OrderedDict()
_CACHE_MAX = 4
_CACHE_LOCK = threading.Lock()


def _key(grid, geometry, wavelet, config, dtype, device, opts):
    samples = np.ascontiguousarray(getattr(wavelet, "samples", wavelet), dtype=np.float64)
    wh = hashlib.sha1(samples.tobytes()).hexdigest()
    g = (grid.nx, grid.nz, float(grid.dx), float(grid.dz))
    geo = (tuple(geometry.sources), tuple(geometry.receivers), float(geometry.dt),
           int(geometry.nt))
    cfg = (config.border_width, config.damping_strength, config.cfl_safety, config.damp_top,
           int(getattr(config, "order", 2)))
    return (g, geo, wh, cfg, str(torch_dtype(dtype)), str(device), tuple(sorted(opts.items())))


def get_propagator(grid, geometry, wavelet, config=SimConfig(), dtype="float64", device=None,
                   **opts) -> Propagator:
    key = _key(grid, geometry, wavelet, config, dtype, device, opts)
    with _CACHE_LOCK:
        prop = _CACHE.get(key)
        if prop is not None:
            _CACHE.move_to_end(key)
            return prop
    prop = Propagator(grid, geometry, wavelet, config, dtype=dtype, device=device, **opts)
    with _CACHE_LOCK:
        _CACHE[key] = prop
        while len(_CACHE) > _CACHE_MAX:
            # dropped, not closed: a caller may still hold it (workspace=...);
            # the handle is released when the last reference goes (__del__)
            _CACHE.popitem(last=False)
    return prop


def clear_cache():
    with _CACHE_LOCK:
        _CACHE.clear()


# ---------------------------------------------------------------------------
# public single-shot solves (seisopt/wavesim.py:354-430)
# ---------------------------------------------------------------------------


@dataclass
class WavefieldHistory:
    """Per-step acceleration on the padded grid (seisopt/wavesim.py:232-246)."""

    accel: np.ndarray
    pad: PadSpec
    grid: object
    dt: float

    def accel_physical(self, n):
        return restrict_to_interior(self.accel[n], self.pad, self.grid)


@dataclass
class AdjointHistory:
    """Per-step adjoint field v_n (seisopt/wavesim.py:249-256)."""

    v: np.ndarray
    pad: PadSpec
    grid: object
    dt: float


def forward_solve(model, wavelet, geometry, source_index, config=SimConfig(), workspace=None,
                  keep_history=True, dtype="float64"):
    """seisopt/wavesim.py:354-378 on the GPU."""
    if wavelet.nt != geometry.nt:
        raise ValueError("wavelet length does not match geometry nt")
    if not (0 <= source_index < geometry.n_sources):
        raise ValueError(f"source_index {source_index} out of range")
    prop = workspace or get_propagator(model.grid, geometry, wavelet, config, dtype)
    with prop._lock:  # model + sweep on one shared handle (see get_propagator)
        prop.set_model(model.m)
        if keep_history:
            g, a = prop.forward_history(source_index)
            hist = WavefieldHistory(accel=a.double().cpu().numpy(), pad=prop.pad,
                                    grid=model.grid, dt=geometry.dt)
        else:
            g = prop.synthetic((source_index, 1))[0]
            hist = None
        g = g.double().cpu().numpy()
    return ShotGather(source_index=source_index, samples=g, dt=geometry.dt), hist


def adjoint_solve(model, adjoint_source, geometry, config=SimConfig(), workspace=None,
                  wavelet=None, dtype="float64"):
    """seisopt/wavesim.py:414-430 on the GPU (v history of one data set)."""
    if adjoint_source.samples.shape != (geometry.nt, geometry.n_receivers):
        raise ValueError("adjoint source shape does not match geometry")
    wav = wavelet if wavelet is not None else np.zeros(geometry.nt)
    prop = workspace or get_propagator(model.grid, geometry, wav, config, dtype)
    with prop._lock:
        prop.set_model(model.m)
        v = prop.adjoint_history(adjoint_source.samples).double().cpu().numpy()
    return AdjointHistory(v=v, pad=prop.pad, grid=model.grid, dt=geometry.dt)


def born_solve(background, reflectivity, wavelet, geometry, source_index, config=SimConfig(),
               workspace=None, dtype="float64"):
    """seisopt/wavesim.py:381-411 on the GPU (lock-step background)."""
    if background.grid != reflectivity.grid:
        raise ValueError("background and reflectivity must share a grid")
    prop = workspace or get_propagator(background.grid, geometry, wavelet, config, dtype)
    with prop._lock:
        prop.set_model(background.m)
        d = prop.born_forward(reflectivity.m_r, (source_index, 1))[0].double().cpu().numpy()
    return ShotGather(source_index=source_index, samples=d, dt=geometry.dt)

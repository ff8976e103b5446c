"""Data-model types consumed by the hot path.

These mirror the reference's public types field for field so that objects built
with either package are interchangeable (the drop-in boundary is duck-typed):

* ``Grid2D``               -- seisopt/grid.py:35-61
* ``VelocityModel``        -- seisopt/grid.py:73-102   (squared slowness m = 1/c^2)
* ``ReflectivityModel``    -- seisopt/grid.py:105-113
* ``AcquisitionGeometry``  -- seisopt/grid.py:116-155
* ``SourceWavelet``        -- seisopt/grid.py:158-176, ``make_ricker`` :179-192
* ``ShotGather``           -- seisopt/wavesim.py:69-89
* ``SimConfig``            -- seisopt/wavesim.py:45-66
* ``EvalCounters``         -- seisopt/counting.py:14-24
* ``ObjectiveEval``        -- seisopt/gradients.py:31-37

Arrays are (nz, nx) C-order, x fastest (seisopt/grid.py:5).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


class StabilityError(Exception):
    """Time step violates the CFL bound (seisopt/wavesim.py:41-42)."""


@dataclass(frozen=True)
class Grid2D:
    nx: int
    nz: int
    dx: float
    dz: float

    def __post_init__(self):
        if self.nx < 3 or self.nz < 3:
            raise ValueError(f"grid must be at least 3x3, got {self.nx}x{self.nz}")
        if self.dx <= 0 or self.dz <= 0:
            raise ValueError("grid spacings must be positive")

    @property
    def shape(self):
        return (self.nz, self.nx)

    @property
    def extent_x(self):
        return (self.nx - 1) * self.dx

    @property
    def extent_z(self):
        return (self.nz - 1) * self.dz


def _field(grid, values, name):
    arr = np.asarray(values, dtype=np.float64)
    if arr.shape != grid.shape:
        raise ValueError(f"{name} shape {arr.shape} does not match grid {grid.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite values")
    return arr


@dataclass(frozen=True)
class VelocityModel:
    grid: Grid2D
    m: np.ndarray

    def __post_init__(self):
        arr = _field(self.grid, self.m, "m")
        if np.any(arr <= 0):
            raise ValueError("squared slowness must be positive everywhere")
        object.__setattr__(self, "m", arr)

    @property
    def velocity(self):
        return 1.0 / np.sqrt(self.m)

    @property
    def c_max(self):
        return float(1.0 / math.sqrt(self.m.min()))

    @property
    def c_min(self):
        return float(1.0 / math.sqrt(self.m.max()))

    @staticmethod
    def from_velocity(grid, c):
        c = np.asarray(c, dtype=np.float64)
        return VelocityModel(grid, 1.0 / (c * c))


@dataclass(frozen=True)
class ReflectivityModel:
    grid: Grid2D
    m_r: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "m_r", _field(self.grid, self.m_r, "m_r"))


@dataclass(frozen=True)
class AcquisitionGeometry:
    sources: tuple
    receivers: tuple
    dt: float
    nt: int

    def __post_init__(self):
        object.__setattr__(self, "sources", tuple((float(x), float(z)) for x, z in self.sources))
        object.__setattr__(self, "receivers",
                           tuple((float(x), float(z)) for x, z in self.receivers))
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.nt < 2:
            raise ValueError("nt must be at least 2")
        if not self.sources or not self.receivers:
            raise ValueError("need at least one source and one receiver")

    @property
    def n_sources(self):
        return len(self.sources)

    @property
    def n_receivers(self):
        return len(self.receivers)

    def validate_against(self, grid):
        for label, pts in (("source", self.sources), ("receiver", self.receivers)):
            for x, z in pts:
                if not (0.0 <= x <= grid.extent_x and 0.0 <= z <= grid.extent_z):
                    raise ValueError(f"{label} ({x}, {z}) outside grid extent "
                                     f"[0, {grid.extent_x}] x [0, {grid.extent_z}]")


@dataclass(frozen=True)
class SourceWavelet:
    samples: np.ndarray
    peak_freq: float
    t0: float

    def __post_init__(self):
        arr = np.asarray(self.samples, dtype=np.float64)
        if arr.ndim != 1:
            raise ValueError("wavelet samples must be 1-D")
        if not np.all(np.isfinite(arr)):
            raise ValueError("wavelet contains non-finite values")
        object.__setattr__(self, "samples", arr)

    @property
    def nt(self):
        return len(self.samples)


def make_ricker(peak_freq, dt, nt, t0=0.0):
    """Ricker wavelet (seisopt/grid.py:179-192)."""
    if peak_freq <= 0 or dt <= 0 or nt < 2:
        raise ValueError("invalid Ricker parameters")
    t = np.arange(nt) * dt - t0
    a = (math.pi * peak_freq) ** 2 * t * t
    return SourceWavelet(samples=(1.0 - 2.0 * a) * np.exp(-a), peak_freq=peak_freq, t0=t0)


@dataclass
class ShotGather:
    source_index: int
    samples: np.ndarray
    dt: float

    def __post_init__(self):
        arr = np.asarray(self.samples, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("gather samples must be 2-D (nt, n_receivers)")
        self.samples = arr

    @property
    def nt(self):
        return self.samples.shape[0]

    @property
    def n_receivers(self):
        return self.samples.shape[1]


@dataclass(frozen=True)
class SimConfig:
    """Sponge geometry and stability margin (seisopt/wavesim.py:45-66).

    ``order`` (2 or 8) selects the spatial stencil: 2 is the reference's
    5-point Laplacian, 8 the BASELINE configs' 8th-order stencil.  It is
    keyword-only in spirit; the first four fields keep the reference order.
    """

    border_width: int = 30
    damping_strength: float = 0.0053
    cfl_safety: float = 0.9
    damp_top: bool = True
    order: int = 2

    def __post_init__(self):
        if self.border_width < 0:
            raise ValueError("border_width must be non-negative")
        if not (0.0 < self.cfl_safety <= 1.0):
            raise ValueError("cfl_safety must lie in (0, 1]")
        if self.damping_strength < 0:
            raise ValueError("damping_strength must be non-negative")
        if self.order not in (2, 8):
            raise ValueError("order must be 2 or 8")


@dataclass
class EvalCounters:
    grad_evals: int = 0
    obj_evals: int = 0

    @property
    def grad_equivalents(self):
        return self.grad_evals + 0.5 * self.obj_evals

    def snapshot(self):
        return EvalCounters(self.grad_evals, self.obj_evals)


@dataclass
class ObjectiveEval:
    value: float
    gradient: np.ndarray
    gradient_eval_count_delta: int = 1

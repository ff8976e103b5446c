"""Data ingress/egress around the hot path, host side.

* ``add_uniform_noise`` / ``measure_snr_db`` -- seisopt/noise.py:12-54: zero-mean
  uniform noise rescaled to an exact dataset SNR, deterministic per seed (same
  generator and draw order as the reference, so the noise is identical).
* ``save_gather`` / ``load_gather`` -- seisopt/wavesim.py:446-492: JSON header +
  sibling little-endian float32 ``.bin``, time-major.
* ``save_grid`` / ``load_grid`` -- seisopt/grid.py:259-323: JSON header + sibling
  float32 ``.bin`` with z fastest; velocity files store m/s.

Files written here are byte-compatible with the reference's.
"""

from __future__ import annotations

import json
import math
import os

import numpy as np

from .model import Grid2D, ReflectivityModel, ShotGather, VelocityModel

GATHER_TAG = "seisopt-gather-v1"
GRID_TAG = "seisopt-grid-v1"
QUANTITIES = ("velocity_mps", "slowness_sq", "reflectivity")


class GridFileError(Exception):
    """Base class of file errors (seisopt/grid.py:23-24)."""


class HeaderMismatchError(GridFileError):
    """Missing / malformed header or wrong format tag (seisopt/grid.py:27-28)."""


class SizeMismatchError(GridFileError):
    """Payload size disagrees with the header (seisopt/grid.py:31-32)."""


# ---------------------------------------------------------------------------
# noise
# ---------------------------------------------------------------------------


def add_uniform_noise(gathers, snr_db: float, seed: int):
    """Noisy copies with 10 log10(P_signal / P_noise) == snr_db over the whole
    dataset (seisopt/noise.py:12-39)."""
    if math.isinf(snr_db) and snr_db > 0:
        return [ShotGather(g.source_index, np.array(g.samples, copy=True), g.dt) for g in gathers]
    power, count = 0.0, 0
    for g in gathers:
        x = np.asarray(g.samples, dtype=np.float64)
        if not np.all(np.isfinite(x)):
            raise ValueError("gather contains non-finite samples")
        power += float(np.sum(x * x))
        count += x.size
    if power == 0.0:
        raise ValueError("cannot set an SNR on all-zero data")
    rng = np.random.default_rng(seed)
    noise = [rng.uniform(-1.0, 1.0, size=np.shape(g.samples)) for g in gathers]
    noise_ms = sum(float(np.sum(n * n)) for n in noise) / count
    gain = math.sqrt((power / count) / (10.0 ** (snr_db / 10.0)) / noise_ms)
    return [ShotGather(g.source_index, g.samples + gain * n, g.dt) for g, n in zip(gathers, noise)]


def measure_snr_db(clean, noisy) -> float:
    """seisopt/noise.py:42-54."""
    ps = pn = 0.0
    for c, n in zip(clean, noisy):
        d = n.samples - c.samples
        ps += float(np.sum(c.samples * c.samples))
        pn += float(np.sum(d * d))
    return float("inf") if pn == 0.0 else 10.0 * math.log10(ps / pn)


# ---------------------------------------------------------------------------
# files
# ---------------------------------------------------------------------------


def _bin_path(path):
    return os.path.splitext(path)[0] + ".bin"


def _write_atomic(path, data: bytes):
    tmp = path + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(data)
    os.replace(tmp, path)


def _header_bytes(header: dict) -> bytes:
    return (json.dumps(header, sort_keys=True, indent=2) + "\n").encode()


def _read_header(path, tag):
    try:
        with open(path, "rb") as fh:
            header = json.loads(fh.read().decode())
    except (json.JSONDecodeError, UnicodeDecodeError) as exc:
        raise HeaderMismatchError(f"{path}: malformed header: {exc}") from exc
    if not isinstance(header, dict) or header.get("format") != tag:
        raise HeaderMismatchError(f"{path}: not a {tag} header")
    return header


def _read_payload(path, nbytes):
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) != nbytes:
        raise SizeMismatchError(f"{path}: expected {nbytes} bytes, got {len(raw)}")
    return raw


def save_gather(gather, path):
    """seisopt/wavesim.py:451-467."""
    header = {"format": GATHER_TAG, "nt": gather.nt, "n_receivers": gather.n_receivers,
              "dt": gather.dt, "source_index": gather.source_index}
    _write_atomic(path, _header_bytes(header))
    _write_atomic(_bin_path(path),
                  np.ascontiguousarray(gather.samples, dtype="<f4").tobytes())


def load_gather(path):
    """seisopt/wavesim.py:470-492."""
    h = _read_header(path, GATHER_TAG)
    try:
        nt, nrec = int(h["nt"]), int(h["n_receivers"])
        dt, src = float(h["dt"]), int(h["source_index"])
    except (KeyError, TypeError, ValueError) as exc:
        raise HeaderMismatchError(f"{path}: incomplete header: {exc}") from exc
    raw = _read_payload(_bin_path(path), nt * nrec * 4)
    data = np.frombuffer(raw, dtype="<f4").reshape(nt, nrec).astype(np.float64)
    return ShotGather(source_index=src, samples=data, dt=dt)


def save_grid(model, path, quantity=None):
    """seisopt/grid.py:259-289 (payload z fastest)."""
    if isinstance(model, ReflectivityModel) or hasattr(model, "m_r"):
        quantity = quantity or "reflectivity"
        values = model.m_r
    elif hasattr(model, "m"):
        quantity = quantity or "velocity_mps"
        values = 1.0 / np.sqrt(model.m) if quantity == "velocity_mps" else model.m
    else:
        raise TypeError(f"cannot save object of type {type(model).__name__}")
    if quantity not in QUANTITIES:
        raise ValueError(f"unknown quantity {quantity!r}")
    g = model.grid
    header = {"format": GRID_TAG, "nx": g.nx, "nz": g.nz, "dx": g.dx, "dz": g.dz,
              "quantity": quantity}
    _write_atomic(path, _header_bytes(header))
    _write_atomic(_bin_path(path), np.ascontiguousarray(np.asarray(values).T,
                                                        dtype="<f4").tobytes())


def load_grid(path):
    """seisopt/grid.py:292-323."""
    h = _read_header(path, GRID_TAG)
    try:
        nx, nz = int(h["nx"]), int(h["nz"])
        dx, dz = float(h["dx"]), float(h["dz"])
        quantity = h["quantity"]
    except (KeyError, TypeError, ValueError) as exc:
        raise HeaderMismatchError(f"{path}: incomplete header: {exc}") from exc
    if quantity not in QUANTITIES:
        raise HeaderMismatchError(f"{path}: unknown quantity {quantity!r}")
    raw = _read_payload(_bin_path(path), nx * nz * 4)
    values = np.frombuffer(raw, dtype="<f4").reshape(nx, nz).T.astype(np.float64)
    grid = Grid2D(nx=nx, nz=nz, dx=dx, dz=dz)
    if quantity == "velocity_mps":
        return VelocityModel.from_velocity(grid, values)
    if quantity == "slowness_sq":
        return VelocityModel(grid, values)
    return ReflectivityModel(grid, values)

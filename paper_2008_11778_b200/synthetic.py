"""Seeded synthetic workloads for the BASELINE configs (BASELINE.json:configs).

The paper's Marmousi benchmark is not available offline; C3-C5 use a seeded
layered-fault generator of the same shape class (3 km x 9 km, water layer over
dipping layers cut by normal faults).  C1 follows the BASELINE text exactly
(linear trend + Gaussian anomaly).  C2 is the standalone AA window.

Every builder returns plain dicts of NumPy arrays and scalars so it can feed
both this package and the reference/oracle.
"""

from __future__ import annotations

import math

import numpy as np

from .model import (AcquisitionGeometry, Grid2D, ReflectivityModel, SimConfig,
                    VelocityModel, make_ricker)


def c1_models():
    """C1: 101x101 at 10 m; c = 2000 -> 3000 m/s with depth; +10% Gaussian
    anomaly (sigma 8 cells) at the grid centre; initial = linear trend."""
    nz = nx = 101
    z = np.arange(nz, dtype=np.float64)[:, None] * np.ones((1, nx))
    trend = 2000.0 + 1000.0 * z / (nz - 1)
    ii, jj = np.mgrid[0:nz, 0:nx]
    r2 = (ii - 50.0) ** 2 + (jj - 50.0) ** 2
    true_c = trend * (1.0 + 0.1 * np.exp(-r2 / (2.0 * 8.0 ** 2)))
    return 1.0 / (true_c * true_c), 1.0 / (trend * trend)


def c1_case(order=8, nt=800):
    """Full C1 problem (BASELINE.json configs[0]).

    Frozen ambiguities: sources at z = 0, x = (i + 1/2) 200 m;
    Ricker t0 = 0.1 s; receivers at z = 2 dx, x = i dx."""
    grid = Grid2D(nx=101, nz=101, dx=10.0, dz=10.0)
    m_true, m_init = c1_models()
    sources = tuple(((i + 0.5) * 200.0, 0.0) for i in range(5))
    receivers = tuple((i * 10.0, 20.0) for i in range(101))
    geom = AcquisitionGeometry(sources, receivers, dt=1e-3, nt=nt)
    wav = make_ricker(10.0, 1e-3, nt, t0=0.1)
    cfg = SimConfig(border_width=20, order=order)
    return dict(grid=grid, true=VelocityModel(grid, m_true), init=VelocityModel(grid, m_init),
                geometry=geom, wavelet=wav, config=cfg, memory=5, iterations=20)


def layered_fault_velocity(nz, nx, dx, seed=0, water_depth=450.0, n_layers=25,
                           v_water=1500.0, v_top=1600.0, v_bottom=4700.0, n_faults=3,
                           max_throw=150.0):
    """Seeded water-over-dipping-layers model cut by normal faults (m/s).

    Geometry is defined in metres, so the same seed gives the same geology at
    15 m (C3/C4) and 3 m (C5) sampling.
    """
    rng = np.random.default_rng(seed)
    depth = (nz - 1) * dx
    width = (nx - 1) * dx
    z = np.arange(nz)[:, None] * dx
    x = np.arange(nx)[None, :] * dx
    # interfaces: dipping planes with slightly varying dip, random thicknesses
    thick = rng.uniform(0.6, 1.4, n_layers)
    thick = thick / thick.sum() * (depth - water_depth) * 1.15
    tops = water_depth + np.concatenate([[0.0], np.cumsum(thick)[:-1]])
    dips = np.tan(np.radians(rng.uniform(-6.0, 6.0) + rng.uniform(-1.5, 1.5, n_layers)))
    vels = np.linspace(v_top, v_bottom, n_layers) + rng.uniform(-60.0, 60.0, n_layers)
    vels = np.clip(vels, v_top, v_bottom)
    # normal faults: plane x = xf + (z - water_depth) * cot(angle); hanging wall
    # (x beyond the plane) is dropped by its throw
    shift = np.zeros((nz, nx))
    for _ in range(n_faults):
        xf = rng.uniform(0.15, 0.85) * width
        ang = np.radians(rng.uniform(55.0, 70.0))
        throw = rng.uniform(0.3, 1.0) * max_throw
        sense = 1.0 if rng.uniform() < 0.5 else -1.0
        plane = xf + sense * (z - water_depth) / np.tan(ang)
        hanging = (x - plane) * sense > 0
        shift = shift + np.where(hanging, throw, 0.0)
    zs = z - shift  # stratigraphic depth
    c = np.full((nz, nx), vels[0])
    for k in range(1, n_layers):
        surface = tops[k] + dips[k] * (x - 0.5 * width)
        c = np.where(zs >= surface, vels[k], c)
    c = np.where(z < water_depth, v_water, c)
    return c


def _smooth(m, sigma):
    from scipy.ndimage import gaussian_filter
    return gaussian_filter(m, sigma=sigma, mode="nearest")  # seisopt/grid.py:228


def layered_case(which="c3", n_shots=None, nt=None, seed=0):
    """C3 / C4 / C5 problem dicts (BASELINE.json configs[2..4])."""
    spec = {
        "c3": dict(nz=201, nx=601, dx=15.0, shots=30, nrec=601, f=5.0, dt=1e-3, nt=4000),
        "c4": dict(nz=201, nx=601, dx=15.0, shots=60, nrec=601, f=15.0, dt=5e-4, nt=6000),
        "c5": dict(nz=1001, nx=3001, dx=3.0, shots=240, nrec=3001, f=20.0, dt=2.5e-4,
                   nt=12000),
    }[which]
    ns = spec["shots"] if n_shots is None else n_shots
    nt = spec["nt"] if nt is None else nt
    nz, nx, dx = spec["nz"], spec["nx"], spec["dx"]
    grid = Grid2D(nx=nx, nz=nz, dx=dx, dz=dx)
    c = layered_fault_velocity(nz, nx, dx, seed=seed)
    m_true = 1.0 / (c * c)
    m_smooth = _smooth(m_true, 12.0)
    width = (nx - 1) * dx
    sources = tuple(((i + 0.5) * width / ns, dx) for i in range(ns))
    rec_x = np.linspace(0.0, width, spec["nrec"])
    receivers = tuple((float(xr), 2.0 * dx) for xr in rec_x)
    geom = AcquisitionGeometry(sources, receivers, dt=spec["dt"], nt=nt)
    wav = make_ricker(spec["f"], spec["dt"], nt, t0=1.2 / spec["f"])
    cfg = SimConfig(border_width=20, order=8)
    out = dict(grid=grid, true=VelocityModel(grid, m_true), init=VelocityModel(grid, m_smooth),
               geometry=geom, wavelet=wav, config=cfg)
    if which == "c4":
        dm = np.zeros_like(m_true)
        dm[1:-1] = 0.5 * (m_true[2:] - m_true[:-2])
        dm[0] = m_true[1] - m_true[0]
        dm[-1] = m_true[-1] - m_true[-2]
        dm = dm / np.max(np.abs(dm)) * 0.05 * float(np.median(m_true))
        out["reflectivity"] = ReflectivityModel(grid, dm)
        out["background"] = out["init"]
    return out


def aa_window_stream(n, count, seed=0, rank=3, dtype=np.float32):
    """C2 stream: (p_k, G_k) pairs, i.i.d. N(0,1) plus a shared smooth rank-3
    component (BASELINE.json configs[1])."""
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, n, dtype=np.float64)
    modes = [np.sqrt(2.0) * np.sin(2.0 * math.pi * (j + 1) * t) for j in range(rank)]
    for _ in range(count):
        pair = []
        for _ in range(2):
            v = rng.standard_normal(n)
            for b in modes:
                v += rng.standard_normal() * b
            pair.append(v.astype(dtype))
        yield pair[0], pair[1]

"""Shared test-case definitions (mirrors tests/golden/make_golden.py inputs)."""

from __future__ import annotations

import os

import numpy as np

from paper_2008_11778_b200 import synthetic
from paper_2008_11778_b200.model import (AcquisitionGeometry, Grid2D, SimConfig,
                                         VelocityModel, make_ricker)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def small_geometry():
    sources = ((333.3, 0.0), (880.0, 47.5))
    receivers = tuple((x, 30.0) for x in np.linspace(0.0, 1180.0, 25)) + (
        (505.0, 37.5), (505.0, 37.5), (1180.0, 780.0))
    return AcquisitionGeometry(sources, receivers, dt=2e-3, nt=300)


def small_case(order, damp_top):
    """The 60x40 case of make_golden.small_setup with the fixture's models."""
    g = golden(f"small_o{order}_{'top' if damp_top else 'free'}")
    grid = Grid2D(nx=60, nz=40, dx=20.0, dz=20.0)
    geom = small_geometry()
    return dict(grid=grid, model=VelocityModel(grid, g["m"]),
                true=VelocityModel(grid, g["m_true"]), geometry=geom,
                wavelet=make_ricker(12.0, 2e-3, 300, t0=0.08),
                config=SimConfig(border_width=10, damp_top=damp_top, order=order), gold=g)


def c1(order):
    case = synthetic.c1_case(order=order)
    case["gold"] = golden(f"c1_o{order}")
    return case


def oracle_setup(model_m, grid, geom, cfg):
    import oracle
    return oracle.Setup(model_m, grid.dx, grid.dz, geom.dt, geom.sources, geom.receivers,
                        border=cfg.border_width, strength=cfg.damping_strength,
                        cfl_safety=cfg.cfl_safety, damp_top=cfg.damp_top, order=cfg.order)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))

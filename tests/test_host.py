"""Host-side logic of the drop-in shim (no GPU): taps, sponge, pads, CFL,
shard assignment, host utilities, synthetic workloads."""

import math

import numpy as np
import pytest

import oracle
from cases import golden, small_case
from paper_2008_11778_b200 import gradients, shards, synthetic, wavesim
from paper_2008_11778_b200.model import (AcquisitionGeometry, Grid2D, ShotGather, SimConfig,
                                         VelocityModel, make_ricker)


@pytest.mark.parametrize("order", [2, 8])
@pytest.mark.parametrize("damp_top", [True, False])
def test_taps_and_sponge_bit_identical(order, damp_top):
    case = small_case(order, damp_top)
    g = case["gold"]
    pad = wavesim.pad_spec(case["config"])
    shape = pad.padded_shape(case["grid"])
    for pts, prefix in ((case["geometry"].receivers, "rec"), (case["geometry"].sources, "src")):
        r, c, w = wavesim.bilinear_taps(pts, case["grid"], pad, shape)
        assert np.array_equal(r, g[prefix + "_rows"])
        assert np.array_equal(c, g[prefix + "_cols"])
        assert np.array_equal(w, g[prefix + "_w"])
    assert np.array_equal(wavesim.damping_mask(case["grid"], case["config"]), g["damp"])


def test_pads_and_fold_are_transposes():
    rng = np.random.default_rng(0)
    grid = Grid2D(nx=7, nz=5, dx=1.0, dz=1.0)
    for top in (True, False):
        pad = wavesim.pad_spec(SimConfig(border_width=3, damp_top=top))
        x = rng.standard_normal(grid.shape)
        y = rng.standard_normal(pad.padded_shape(grid))
        pads = (pad.top, pad.bottom, pad.left, pad.right)
        lhs = float(np.sum(wavesim.extend_to_pad(x, pad) * y))
        rhs = float(np.sum(x * oracle.fold_pad(y, pads, grid.nz, grid.nx)))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
        assert np.array_equal(wavesim.restrict_to_interior(wavesim.extend_to_pad(x, pad), pad,
                                                           grid), x)


def test_cfl_bounds():
    grid = Grid2D(nx=10, nz=10, dx=20.0, dz=20.0)
    m = VelocityModel.from_velocity(grid, np.full(grid.shape, 2000.0))
    assert abs(wavesim.cfl_check(m) - 20.0 / (2000.0 * math.sqrt(2.0))) < 1e-15
    assert abs(wavesim.cfl_check(m, order=8) / wavesim.cfl_check(m) - 0.78439) < 1e-4
    assert abs(wavesim.CFL8_FACTOR - oracle.CFL8_FACTOR) < 1e-15


@pytest.mark.parametrize("n,world", [(30, 8), (5, 2), (240, 8), (60, 7), (3, 3)])
def test_shard_bounds(n, world):
    got = [shards.shard_bounds(n, world, r) for r in range(world)]
    assert got[0][0] == 0
    for (s0, c0), (s1, _) in zip(got, got[1:]):
        assert s1 == s0 + c0
    assert sum(c for _, c in got) == n
    assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_misfit_known_answers():
    dt = 0.004
    z = np.zeros((5, 3))
    e = z.copy()
    e[2, 1] = 1.0
    s = [ShotGather(0, e, dt)]
    o = [ShotGather(0, z, dt)]
    assert gradients.misfit_l2(s, o) == 0.5 * dt
    assert gradients.misfit_l2(o, o) == 0.0
    assert gradients.misfit_l2(s, o) == oracle.misfit_l2([e], [z], dt)
    with pytest.raises(ValueError):
        gradients.misfit_l2(s, [ShotGather(0, np.zeros((4, 3)), dt)])
    r = gradients.adjoint_source(s, o)
    assert np.array_equal(r[0].samples, e)


def test_laplacian_filter():
    assert np.all(gradients.laplacian_filter(np.full((4, 5), 3.0)) == 0.0)
    x = np.zeros((5, 5))
    x[2, 2] = 1.0
    y = gradients.laplacian_filter(x)
    assert y[2, 2] == 4.0 and y[1, 2] == -1.0 and y[2, 3] == -1.0


def test_pairwise_sum_matches_oracle():
    rng = np.random.default_rng(2)
    arrs = [rng.standard_normal((3, 4)) for _ in range(7)]
    assert np.array_equal(gradients.pairwise_sum(arrs), oracle.tree_sum(arrs))


def test_synthetic_workloads():
    c = synthetic.layered_fault_velocity(201, 601, 15.0, seed=0)
    assert c.shape == (201, 601)
    assert np.all(c[:30] == 1500.0)                       # 450 m water layer
    assert 1600.0 <= c[30:].min() and c.max() <= 4700.0
    assert len(np.unique(c[30:])) >= 20                    # many layers
    c2 = synthetic.layered_fault_velocity(201, 601, 15.0, seed=0)
    assert np.array_equal(c, c2)                           # seeded
    case = synthetic.layered_case("c3")
    g = case["geometry"]
    assert g.n_sources == 30 and g.n_receivers == 601 and g.nt == 4000
    assert case["config"].order == 8 and case["config"].border_width == 20
    m1, m0 = synthetic.c1_models()
    assert m1.shape == (101, 101) and np.all(m1 <= m0 + 1e-20)
    p, gg = next(synthetic.aa_window_stream(1000, 1))
    assert p.dtype == np.float32 and p.shape == (1000,)


def test_model_types_validate():
    grid = Grid2D(nx=5, nz=4, dx=1.0, dz=1.0)
    with pytest.raises(ValueError):
        VelocityModel(grid, -np.ones(grid.shape))
    with pytest.raises(ValueError):
        AcquisitionGeometry((), ((0.0, 0.0),), 1e-3, 10)
    w = make_ricker(10.0, 1e-3, 201, t0=0.1)
    assert abs(w.samples.max() - 1.0) < 1e-12
    with pytest.raises(ValueError):
        SimConfig(order=4)


def test_reference_types_are_accepted(reference_available):
    """The shim is duck-typed: the reference's own objects work as inputs."""
    if not reference_available:
        pytest.skip("reference not mounted")
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from seisopt.grid import AcquisitionGeometry as RG, Grid2D as RGrid
    grid = RGrid(nx=60, nz=40, dx=20.0, dz=20.0)
    geo = RG(((333.3, 0.0),), ((100.0, 30.0),), 2e-3, 10)
    pad = wavesim.pad_spec(SimConfig(border_width=10))
    r, c, w = wavesim.bilinear_taps(geo.receivers, grid, pad, pad.padded_shape(grid))
    assert r.shape == (4, 1)

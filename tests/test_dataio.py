"""Noise and file formats (host): semantics and byte compatibility with the
reference (compared against seisopt itself when it is mounted)."""

import math
import os
import sys

import numpy as np
import pytest

from paper_2008_11778_b200 import dataio
from paper_2008_11778_b200.model import Grid2D, ReflectivityModel, ShotGather, VelocityModel


def _gathers(seed=0):
    rng = np.random.default_rng(seed)
    return [ShotGather(s, rng.standard_normal((50, 7)), 1e-3) for s in range(3)]


def test_noise_exact_snr_and_determinism():
    g = _gathers()
    n1 = dataio.add_uniform_noise(g, 0.55, 1234)
    n2 = dataio.add_uniform_noise(g, 0.55, 1234)
    assert abs(dataio.measure_snr_db(g, n1) - 0.55) < 1e-9
    assert all(np.array_equal(a.samples, b.samples) for a, b in zip(n1, n2))
    same = dataio.add_uniform_noise(g, math.inf, 1)
    assert all(np.array_equal(a.samples, b.samples) for a, b in zip(g, same))
    assert dataio.measure_snr_db(g, same) == math.inf
    with pytest.raises(ValueError):
        dataio.add_uniform_noise([ShotGather(0, np.zeros((4, 2)), 1e-3)], 3.0, 0)


def test_file_round_trips(tmp_path):
    g = _gathers()[1]
    p = str(tmp_path / "shot.json")
    dataio.save_gather(g, p)
    r = dataio.load_gather(p)
    assert r.source_index == 1 and r.dt == g.dt
    assert np.array_equal(r.samples, g.samples.astype(np.float32).astype(np.float64))
    grid = Grid2D(nx=6, nz=4, dx=10.0, dz=5.0)
    c = 1500.0 + 100.0 * np.arange(24, dtype=np.float64).reshape(4, 6)
    vm = VelocityModel.from_velocity(grid, c)
    q = str(tmp_path / "model.json")
    dataio.save_grid(vm, q)
    back = dataio.load_grid(q)
    assert back.grid == grid and np.allclose(back.velocity, c, rtol=1e-7)
    dataio.save_grid(vm, q, quantity="slowness_sq")
    assert np.allclose(dataio.load_grid(q).m, vm.m, rtol=1e-7)
    rm = ReflectivityModel(grid, np.arange(24.0).reshape(4, 6))
    dataio.save_grid(rm, q)
    assert np.array_equal(dataio.load_grid(q).m_r, rm.m_r)
    with open(q.replace(".json", ".bin"), "ab") as fh:
        fh.write(b"xx")
    with pytest.raises(dataio.SizeMismatchError):
        dataio.load_grid(q)
    with open(q, "w") as fh:
        fh.write("{not json")
    with pytest.raises(dataio.HeaderMismatchError):
        dataio.load_grid(q)


def test_byte_compatible_with_reference(tmp_path, reference_available):
    if not reference_available:
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from seisopt import noise as rnoise
    from seisopt import wavesim as rws
    from seisopt import grid as rgrid
    g = _gathers(3)
    ref = rnoise.add_uniform_noise([rws.ShotGather(x.source_index, x.samples, x.dt) for x in g],
                                   2.0, 77)
    mine = dataio.add_uniform_noise(g, 2.0, 77)
    assert all(np.array_equal(a.samples, b.samples) for a, b in zip(ref, mine))
    for name, saver, obj in (("g", rws.save_gather, rws.ShotGather(0, g[0].samples, 1e-3)),):
        saver(obj, str(tmp_path / "ref.json"))
        dataio.save_gather(g[0], str(tmp_path / "mine.json"))
        for ext in (".json", ".bin"):
            assert (tmp_path / ("ref" + ext)).read_bytes() == (tmp_path / ("mine" + ext)).read_bytes()
    rg = rgrid.Grid2D(nx=6, nz=4, dx=10.0, dz=5.0)
    c = 1500.0 + 100.0 * np.arange(24, dtype=np.float64).reshape(4, 6)
    rgrid.save_grid(rgrid.VelocityModel.from_velocity(rg, c), str(tmp_path / "rm.json"))
    dataio.save_grid(VelocityModel.from_velocity(Grid2D(nx=6, nz=4, dx=10.0, dz=5.0), c),
                     str(tmp_path / "mm.json"))
    for ext in (".json", ".bin"):
        assert (tmp_path / ("rm" + ext)).read_bytes() == (tmp_path / ("mm" + ext)).read_bytes()

"""Multi-rank shot sharding on CPU (gloo, world_size 2): each rank computes
its shard's gradient (oracle as the per-rank compute stand-in) and the single
all-reduce of (gradient, misfit) reproduces the full gradient."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from cases import oracle_setup, small_case
        from paper_2008_11778_b200 import shards
        case = small_case(8, True)
        g = case["gold"]
        geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
        sh = shards.ShotShard.from_env(geom.n_sources)
        st = oracle_setup(g["m"], grid, geom, cfg)
        ids = range(sh.shot0, sh.shot0 + sh.count)
        val, grad, _ = oracle.fwi_gradient(st, [g["obs"][i] for i in ids], wav.samples,
                                           geom.nt, shots=ids)
        t = torch.as_tensor(grad.copy())
        tot = sh.allreduce_value_grad(val, t)
        t32 = torch.as_tensor(grad.astype(np.float32))
        tot32 = sh.allreduce_value_grad(val, t32)
        q.put((rank, sh.shot0, sh.count, tot, t.numpy(), tot32))
    finally:
        dist.destroy_process_group()


def test_two_rank_gradient_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert [(o[1], o[2]) for o in out] == [(0, 1), (1, 1)]
    from cases import small_case
    g = small_case(8, True)["gold"]
    for _, _, _, tot, grad, tot32 in out:
        assert abs(tot - float(g["value"])) <= 1e-12 * float(g["value"])
        assert np.linalg.norm(grad - g["grad"]) <= 1e-12 * np.linalg.norm(g["grad"])
        assert abs(tot32 - float(g["value"])) <= 1e-12 * float(g["value"])
    assert np.array_equal(out[0][4], out[1][4])


def _worker3(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from cases import c1, oracle_setup
        from paper_2008_11778_b200 import shards
        case = c1(8)
        g = case["gold"]
        geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
        sh = shards.ShotShard.from_env(geom.n_sources)
        ids = list(range(sh.shot0, sh.shot0 + sh.count))
        st_true = oracle_setup(g["m_true"], grid, geom, cfg)
        obs = oracle.fwi_synthetic(st_true, wav.samples, geom.nt, shots=ids)
        st = oracle_setup(g["m_init"], grid, geom, cfg)
        val, grad, _ = oracle.fwi_gradient(st, obs, wav.samples, geom.nt, shots=ids)
        t = torch.as_tensor(grad.copy())
        tot = sh.allreduce_value_grad(val, t)
        q.put((rank, sh.shot0, sh.count, tot, t.numpy()))
    finally:
        dist.destroy_process_group()


def test_three_rank_uneven_shards():
    """C1's 5 shots over 3 ranks (2, 2, 1): uneven contiguous blocks
    (seisopt/gradients.py:91-95, :150-152 sums all shots) reduce to the
    reference's 5-shot value and gradient."""
    from paper_2008_11778_b200 import shards
    assert [shards.shard_bounds(30, 8, r)[1] for r in range(8)] == [4, 4, 4, 4, 4, 4, 3, 3]
    assert [shards.shard_bounds(240, 8, r) for r in (0, 7)] == [(0, 30), (210, 30)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert [(o[1], o[2]) for o in out] == [(0, 2), (2, 2), (4, 1)]
    from cases import golden
    g = golden("c1_o8")
    for _, _, _, tot, grad in out:
        assert abs(tot - float(g["value"])) <= 1e-11 * float(g["value"])
        assert np.linalg.norm(grad - g["grad"]) <= 1e-11 * np.linalg.norm(g["grad"])
    assert np.array_equal(out[0][4], out[1][4]) and np.array_equal(out[0][4], out[2][4])

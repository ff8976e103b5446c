"""Sharded objective on the GPU: two ranks own disjoint shot blocks of the C1
survey, run them through libseisgpu on cuda:0 and join with one all-reduce of
(gradient, misfit) per gradient (gloo here: one GPU is available, and gloo
keeps the two ranks' kernels independent of each other; bench.py uses NCCL).
The reduced misfit / gradient must be the reference's (fp64, 1e-10), and
device-resident AA iterations driven by it must stay identical on both
ranks (the replicated optimizer state)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from cases import c1, oracle_setup
        from paper_2008_11778_b200 import anderson, gradients, shards
        torch.cuda.set_device(0)
        case = c1(8)
        g = case["gold"]
        geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
        st = oracle_setup(g["m_true"], grid, geom, cfg)
        obs = np.stack(oracle.fwi_synthetic(st, wav.samples, geom.nt, threads=5))
        sh = shards.ShotShard.from_env(geom.n_sources)
        obj = gradients.FwiObjective(grid, obs, wav, geom, cfg, dtype="float64", shard=sh)
        p0 = g["m_init"].ravel()
        val, grad = obj.value_and_grad(p0)
        mis = obj.value(p0)
        res = anderson.minimize_aa(obj, p0, memory=5, max_iters=3)
        rows = np.array([r.objective for r in res.report.rows])
        q.put((rank, sh.shot0, sh.count, val, np.asarray(grad), mis, rows,
               np.asarray(res.p)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_gradient_and_aa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from cases import c1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert len(o) > 2, o
    for p in procs:
        assert p.exitcode == 0
    out.sort(key=lambda o: o[0])
    assert [(o[1], o[2]) for o in out] == [(0, 3), (3, 2)]
    g = c1(8)["gold"]
    ref_v, ref_g = float(g["value"]), g["grad"].ravel()
    for _, _, _, val, grad, mis, _, _ in out:
        assert abs(val - ref_v) <= 1e-10 * ref_v
        assert abs(mis - ref_v) <= 1e-10 * ref_v
        assert np.linalg.norm(grad - ref_g) <= 1e-10 * np.linalg.norm(ref_g)
    # replicated optimizer state: both ranks took the same iterates
    assert np.array_equal(out[0][6], out[1][6])
    assert np.array_equal(out[0][7], out[1][7])
    assert np.allclose(out[0][6], g["aa_rows"][:len(out[0][6]), 1], rtol=1e-9)

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


def _aa_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import golden
        from paper_2008_11778_b200 import anderson, shards
        torch.cuda.set_device(0)
        out = {}
        for name in ("aa_window", "aa_illcond"):
            g = golden(name)
            n, memory = int(g["n"]), int(g["memory"])
            i0, cnt = shards.shard_bounds(n, world, rank)
            win = anderson.AAWindow(cnt, memory, dtype="float64", shard_group=True)
            rows = []
            for k in range(len(g["ps"])):
                win.push(g["ps"][k][i0:i0 + cnt], g["gs"][k][i0:i0 + cnt])
                if win.m_k:
                    w = anderson.aa_weights(win)
                    step = np.asarray(anderson.aa_step(win, 1.0, w))
                    rows.append((win.m_k, w.gamma.copy(), w.alpha.copy(), w.residual_norm,
                                 step, win.qr_info()[0]))
                else:
                    rows.append((0, None, None, None, np.asarray(anderson.aa_step(win)), False))
            out[name] = rows
        q.put((rank, out))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_n_sharded_aa_window():
    """the standalone AA step on several GPUs shards N.  Two ranks
    (gloo, both on cuda:0) each hold half of the N-vectors; the window sums
    its inner products over the ranks (sg_aa_set_reducer).  Every rank must
    reproduce the reference's window sizes, gamma, alpha and residual norms
    (tests/golden/aa_window.npz; aa_illcond.npz exercises the sharded device
    QR fallback), hold identical weights, and own its slice of the
    reference's next iterate."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from cases import golden
    from paper_2008_11778_b200 import shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_aa_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for o in res:
        assert isinstance(o[1], dict), o
    res.sort(key=lambda o: o[0])
    for name, tol in (("aa_window", 1e-10), ("aa_illcond", 1e-6)):
        g = golden(name)
        n = int(g["n"])
        r0, r1 = res[0][1][name], res[1][1][name]
        used_qr = 0
        for k in range(len(g["ps"])):
            mk = int(g["m_k"][k])
            assert r0[k][0] == r1[k][0] == mk, (name, k)
            full = np.concatenate([r0[k][4], r1[k][4]])
            assert full.shape == (n,)
            assert np.linalg.norm(full - g["step1"][k]) <= tol * np.linalg.norm(g["step1"][k])
            if not mk:
                continue
            # identical weights on both ranks (replicated host algebra on
            # identical reduced sums)
            assert np.array_equal(r0[k][1], r1[k][1]) and r0[k][3] == r1[k][3]
            gam = g["gamma"][k][:mk]
            assert np.linalg.norm(r0[k][1] - gam) <= tol * max(np.linalg.norm(gam), 1e-300)
            assert abs(r0[k][3] - float(g["resid"][k])) <= max(tol, 1e-7) * float(g["resid"][k])
            if "alpha" in g.files:
                assert np.allclose(r0[k][2], g["alpha"][k][:mk + 1], rtol=1e-10, atol=1e-12)
            used_qr += bool(r0[k][5])
        if name == "aa_illcond":
            assert used_qr >= 5
    # the shard sizes the workers used
    assert shards.shard_bounds(int(golden("aa_window")["n"]), 2, 1)[1] > 0

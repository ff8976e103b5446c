"""Benchmark: FWI gradient throughput of the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c1|c5|c2]
                    [--impl ours|reference]

Workload (default, BASELINE.json configs[2] = "C3"): one complete FWI gradient
per step -- 30 shots, 201x601 grid (241x641 padded), nt 4000, 8th-order
stencil, fp32, 20-cell sponge: forward sweep with history store, residual +
misfit, adjoint sweep with fused imaging, image reduction, fold, and (N > 1)
one all-reduce.  Shots are sharded over the N ranks in contiguous blocks.
C3/C4 scale weakly (each rank owns the config's shot count; the survey has
30*N / 60*N evenly spaced shots); C5 is the fixed 240-shot survey split over
the ranks (strong); --scaling overrides.  Synthetic seeded layered-fault model (the paper's Marmousi
is not available offline).

metric: Gcell-updates/s = 2 * shots * nt * padded cells per gradient (forward +
adjoint stencil sweeps; recompute sweeps of checkpoint mode are not counted)
divided by the device time, max over ranks.  gradients/s is reported beside.

--impl reference times the reference algorithm on the host CPU (the oracle
port, oracle/seisopt_oracle.py, NumPy, reference operation order; the
reference itself is pure Python and cannot be compiled) on a bounded sample of
the same workload with all host threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "wave-stencil Gcell-updates/s (FWI gradient, fwd+adj)"
UNIT = "Gcell-updates/s"
FALLBACK_HBM = 6650.0


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        util = [float(r[7]) for r in self.rows if len(r) > 7 and r[7].isdigit()]
        loaded = [s for s, u in zip(sm, util) if u >= 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def build_case(config, n_shots=None):
    from paper_2008_11778_b200 import synthetic
    if config == "c1":
        case = synthetic.c1_case(order=8)
        case["dtype"] = "float64"
        return case
    case = synthetic.layered_case(config, n_shots=n_shots)
    case["dtype"] = "float32"
    return case


BASE_SHOTS = {"c1": 5, "c3": 30, "c4": 60, "c5": 240}


def scaling_mode(args):
    """C3/C4: weak (each rank owns the config's full shot set, the survey grows
    with N).  C5 is quoted as a fixed 240-shot survey sharded over 1..8 GPUs
    (strong); C1 is a parity case (strong, replicas of 5 shots)."""
    if args.scaling != "auto":
        return args.scaling
    return "weak" if args.config in ("c3", "c4") else "strong"


def total_shots(args, world):
    base = BASE_SHOTS[args.config]
    return base * world if scaling_mode(args) == "weak" else base


def padded_cells(case):
    cfg, grid = case["config"], case["grid"]
    top = cfg.border_width if cfg.damp_top else 0
    return (grid.nz + top + cfg.border_width) * (grid.nx + 2 * cfg.border_width)


def cpu_sample(case, threads, shots, nt):
    """Reference algorithm (oracle port, NumPy) on a bounded sample: `shots`
    shots, first `nt` steps, full C3 grid.  Returns (seconds, cell-updates)."""
    import oracle
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    ids = list(np.linspace(0, geom.n_sources - 1, shots).round().astype(int))
    src = [geom.sources[i] for i in ids]
    st = oracle.Setup(case["init"].m, grid.dx, grid.dz, geom.dt, src, geom.receivers,
                      border=cfg.border_width, strength=cfg.damping_strength,
                      cfl_safety=cfg.cfl_safety, damp_top=cfg.damp_top, order=cfg.order)
    amp = wav.samples[:nt]
    rng = np.random.default_rng(0)
    obs = [rng.standard_normal((nt, geom.n_receivers)) * 1e-3 for _ in ids]
    t0 = time.perf_counter()
    oracle.fwi_gradient(st, obs, amp, nt, threads=threads)
    dt = time.perf_counter() - t0
    cells = 2.0 * shots * nt * st.shape[0] * st.shape[1]
    return dt, cells


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    case = build_case(args.config)
    cores = os.cpu_count() or 1
    shots = min(case["geometry"].n_sources, cores)
    nt = {"c1": 800, "c3": 250, "c4": 150, "c5": 20}.get(args.config, 200)
    for _ in range(args.warmup):
        cpu_sample(case, cores, shots, max(4, nt // 10))
    rates, times = [], []
    for _ in range(args.steps):
        dt, cells = cpu_sample(case, cores, shots, nt)
        rates.append(cells / dt / 1e9)
        times.append(dt)
    value = statistics.median(rates)
    sample = (f"{shots} shots x {nt} of {case['geometry'].nt} steps on the full "
              f"{case['grid'].nz}x{case['grid'].nx} grid per step, fwi_gradient (fwd+hist, "
              f"adjoint+imaging), threads={cores}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": scaling_mode(args), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(args.config), "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_reference_c2(args):
    import oracle
    rank, _, _ = env_rank()
    if rank != 0:
        return 0
    nc, m, n = 5_000_000, 10, 50_000_000
    rng = np.random.default_rng(0)
    wo = oracle.AAWindowOracle(nc, m)
    vecs = [(rng.standard_normal(nc), rng.standard_normal(nc))
            for _ in range(m + 1 + args.warmup + args.steps)]
    for k in range(m + 1 + args.warmup):
        wo.push(*vecs[k])
    times = []
    for k in range(m + 1 + args.warmup, len(vecs)):
        t0 = time.perf_counter()
        wo.push(*vecs[k])
        oracle.aa_step(wo, 1.0, oracle.aa_weights(wo))
        times.append((time.perf_counter() - t0) * 1e3 * (n / nc))
    v = statistics.median(times)
    sample = f"AAWindow push+weights+step at N={nc} (scaled x{n // nc} to N=5e7), m={m}"
    print(json.dumps({"impl": "reference", "metric": "AA mixing step time (push + weights + step)",
                      "value": v, "unit": "ms/iteration", "n_gpus": args.gpus,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": v,
                      "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
                      "dtype": "f64", "data": "synthetic",
                      "config": {"workload": "C2 standalone AA mixing step", "sample": sample},
                      "cpu_baseline": {"value": v, "unit": "ms/iteration",
                                       "cores": os.cpu_count() or 1, "kind": "port",
                                       "sample": sample},
                      "e2e": {"value": v, "unit": "ms/iteration", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)
    return 0


def workload_name(config):
    return {
        "c1": "C1 FWI gradient: 101x101, 5 shots, nt 800, 8th order, fp64",
        "c3": "C3 FWI gradient: layered-fault 201x601 @15 m, 30 shots, 601 rec, nt 4000, "
              "8th order, fp32",
        "c4": "C4 FWI-style gradient on the LSRTM grid: 201x601, 60 shots, nt 6000, fp32",
        "c5": "C5 FWI gradient: 1001x3001 @3 m, 240 shots, 3001 rec, nt 12000, fp32",
    }.get(config, config)


def run_lsrtm(args):
    """C4 (configs[3]): one LSRTM gradient per step -- Born forward (background
    and scattered fields in lock-step), residual, Born adjoint with imaging --
    60 shots, 201x601, nt 6000, fp32.  The 60 background histories (233 GB)
    do not fit in HBM, so the background is recomputed (checkpoints)."""
    import torch
    import torch.distributed as dist

    from paper_2008_11778_b200 import _lib, gradients, shards
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    case = build_case("c4", total_shots(args, world))
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    S, nt = geom.n_sources, geom.nt
    shard = shards.ShotShard.from_env(S) if world > 1 else None
    kern = gradients.BornKernel(case["background"], wav, geom, cfg, dtype="float32", device=dev,
                                shard=shard)
    d_r = kern.forward_device(case["reflectivity"].m_r)      # observed Born data (untimed)
    obj = gradients.LsrtmObjective(kern, d_r)
    p_dev = torch.zeros(grid.nz * grid.nx, device=dev, dtype=torch.float32)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        obj.value_and_grad(p_dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0.record()
        for _ in range(args.steps):
            val, grad = obj.value_and_grad(p_dev)
        e1.record()
        barrier()
    launches = _lib.launch_count() - l0
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    C = padded_cells(case)
    cells = 3.0 * S * nt * C  # background + scattered + adjoint sweeps per gradient
    p_host = np.zeros(grid.nz * grid.nx)
    obj.value_and_grad(p_host)  # untimed: the host path's first-use allocations
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        obj.value_and_grad(p_host)
    barrier()
    e2e_s = time.perf_counter() - t0
    if rank == 0:
        q = kern.ws.query()
        print(json.dumps({
            "metric": "LSRTM wave-stencil Gcell-updates/s (Born fwd + adjoint)",
            "value": cells * args.steps / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": scaling_mode(args), "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C4 LSRTM gradient: layered-fault 201x601 @15 m, 60 shots, "
                                   "601 rec, nt 6000, 15 Hz, 8th order, fp32",
                       "recon": q["recon"], "shots_per_launch": q["batch"],
                       "cached_background": kern.cached},
            "gradients_per_s": args.steps / (ms / 1e3), "misfit": val,
            "e2e": {"value": cells * args.steps / e2e_s / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": p_host.nbytes, "d2h_bytes_per_step": p_host.nbytes + 8},
            "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": None}),
            flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2008_11778_b200 import _lib, gradients, shards
    from paper_2008_11778_b200.model import VelocityModel

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    case = build_case(args.config, total_shots(args, world))
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    S, nt = geom.n_sources, geom.nt
    shard = shards.ShotShard.from_env(S) if world > 1 else None
    # observed data: forward model of the true model on this rank's shots (untimed)
    from paper_2008_11778_b200.wavesim import Propagator
    tmp = Propagator(grid, geom, wav, cfg, dtype=case["dtype"], device=dev)
    tmp.set_model(case["true"].m)
    s0, cnt = (shard.shot0, shard.count) if shard else (0, S)
    obs_local = tmp.synthetic((s0, cnt))
    tmp.close()
    del tmp
    obs_full = torch.zeros((S, nt, geom.n_receivers), dtype=obs_local.dtype, device=dev)
    obs_full[s0:s0 + cnt] = obs_local
    del obs_local
    # the sweep buffers may take 80 % of what is free once the observed data
    # are resident (C5: boundary-saving batches of ~12 shots)
    budget = 0.0
    if args.config == "c5":
        budget = 0.8 * (torch.cuda.mem_get_info(dev)[0] - obs_full.numel() * obs_full.element_size())
    obj = gradients.FwiObjective(grid, obs_full, wav, geom, cfg, dtype=case["dtype"],
                                 device=dev, shard=shard, mem_budget_bytes=budget)
    del obs_full
    torch.cuda.empty_cache()
    p_host = np.ascontiguousarray(case["init"].m.ravel())
    p_dev = torch.as_tensor(p_host, device=dev, dtype=obj.prop.tdtype)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        obj.value_and_grad(p_dev)
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            val, grad = obj.value_and_grad(p_dev)
        e1.record(stream)
        barrier()
    launches = _lib.launch_count() - l0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    C = padded_cells(case)
    cells_per_grad = 2.0 * S * nt * C
    value = cells_per_grad * args.steps / (ms / 1e3) / 1e9
    grads_per_s = args.steps / (ms / 1e3)

    # e2e through the public API with host buffers (numpy model in, numpy
    # gradient out): H2D of the model and D2H of the gradient every step
    # (one untimed call first: the host path's first-use allocations)
    obj.value_and_grad(p_host)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        val_h, grad_h = obj.value_and_grad(p_host)
    barrier()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    e2e_value = cells_per_grad * args.steps / e2e_s / 1e9
    nbytes = p_host.nbytes

    # roofline of the dominant kernel (adjoint step + imaging), timed live with
    # CUDA events on the launching stream; the step launches run as the sweep
    # runs them (two concurrent half-batch chains), so the time is per step of
    # the whole batch and the bytes those of all its shots
    prop = obj.prop
    local_shots = shard.count if shard else S
    es = prop.esz
    q = prop.query()
    launch_shots = min(local_shots, q["batch"])         # shots per step launch
    reps = 100 if launch_shots * C < 2e7 else 20
    if q["recon"] == "boundary":
        # band-storing forward (stencil 4s; the sponge-frame store is <6 % of
        # cells, not counted) and the fused reverse-forward + adjoint step
        # (two stencil updates 8s + imaging 3s)
        ms_fwd = prop.time_step_kernel(6, launch_shots, reps=reps)
        ms_adj = prop.time_step_kernel(5, launch_shots, reps=reps)
        bytes_fwd = launch_shots * C * (4 * es)
        bytes_adj = launch_shots * C * (8 * es + 3 * es)
        names = ("forward_band_step", "reverse_adjoint_step")
    else:
        ms_fwd = prop.time_step_kernel(0, launch_shots, reps=reps)
        ms_adj = prop.time_step_kernel(1, launch_shots, reps=reps)
        bytes_fwd = launch_shots * C * (4 * es + es)       # stencil 4s + history store s
        bytes_adj = launch_shots * C * (4 * es + 3 * es)   # stencil 4s + imaging 3s
        names = ("forward_step", "adjoint_step")
    peak, peak_src = peaks()
    dom = (names[1], ms_adj, bytes_adj) if ms_adj * 1.0 >= ms_fwd else \
        (names[0], ms_fwd, bytes_fwd)
    achieved = dom[2] / (dom[1] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath)).get(args.config, {})
            traffic = tr.get(dom[0])
            if traffic is not None and tr.get("per_shot"):
                traffic *= launch_shots
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        shots = min(S, cores)
        nts = {"c1": 800, "c3": 250, "c4": 150, "c5": 20}.get(args.config, 200)
        dt, cells = cpu_sample(case, cores, shots, nts)
        cpu = {"value": cells / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"oracle fwi_gradient, {shots} shots x {nts} steps of the same grid, "
                         f"threads={cores}, {dt:.1f} s"}
    if rank == 0:
        if q["recon"] == "full":
            l2 = ("inputs larger than L2 (history store %.1f GB per rank)"
                  % (local_shots * nt * C * es / 1e9))
        elif q["recon"] == "boundary":
            l2 = ("inputs larger than L2 (boundary saving; %.1f GB of sponge-frame store per batch)"
                  % (q["device_bytes"] / 1e9))
        else:
            l2 = ("inputs larger than L2 (checkpointed; %.1f GB of fields per launch)"
                  % (launch_shots * C * es * 5 / 1e9))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": scaling_mode(args), "vs_baseline": None,
            "dtype": "f32" if es == 4 else "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "shots": S,
                       "shots_per_rank": local_shots, "nt": nt,
                       "padded_cells": C, "order": cfg.order, "recon": q["recon"],
                       "shots_per_batch": q["batch"], "chains": prop.chains(q["batch"]),
                       "l2": l2},
            "gradients_per_s": grads_per_s,
            "misfit": val,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes + 8, "gradients_per_s": args.steps / e2e_s},
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved,
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         # ncu DRAM bytes of the step / its live time: the HBM
                         # actually moved (C3 fields stay in L2, so < achieved)
                         "traffic_gbs": (traffic / (dom[1] / 1e3) / 1e9) if traffic else None,
                         "shots_per_step": launch_shots,
                         "chains": prop.chains(launch_shots),
                         "bytes_per_step": dom[2], "ms_per_step": dom[1],
                         "forward_ms_per_step": ms_fwd, "adjoint_ms_per_step": ms_adj},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def aa_stream_torch(n, count, seed, dev, dtype):
    """C2 stream on the device: N(0,1) vectors plus a shared smooth rank-3
    component (BASELINE.json configs[1]); same recipe as synthetic.aa_window_stream."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    t = torch.linspace(0.0, 1.0, n, device=dev, dtype=torch.float64)
    modes = [np.sqrt(2.0) * torch.sin(2.0 * np.pi * (j + 1) * t) for j in range(3)]
    out = []
    for _ in range(count):
        pair = []
        for _ in range(2):
            v = torch.randn(n, generator=g, device=dev, dtype=torch.float64)
            c = torch.randn(3, generator=g, device=dev, dtype=torch.float64)
            for j in range(3):
                v += c[j] * modes[j]
            pair.append(v.to(dtype))
        out.append(pair)
    return out


def run_c2(args):
    """Standalone AA mixing step (configs[1]): N = 5e7 fp32, m = 10; one step =
    push (fused residual-difference + Gram row pass) + host m x m solve +
    recombination, window full and sliding."""
    import torch

    from paper_2008_11778_b200 import _lib, anderson
    rank, world, local = env_rank()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, m = 50_000_000, 10
    total = m + 1 + args.warmup + args.steps
    stream = aa_stream_torch(n, total, 0, dev, torch.float32)
    win = anderson.AAWindow(n, m, dtype="float32", device=dev)
    out = torch.empty(n, device=dev, dtype=torch.float32)
    for k in range(m + 1 + args.warmup):
        win.push(*stream[k])
        if win.m_k:
            anderson.aa_step(win, weights=anderson.aa_weights(win), out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        e0.record()
        for k in range(m + 1 + args.warmup, total):
            win.push(*stream[k])
            w = anderson.aa_weights(win)
            anderson.aa_step(win, weights=w, out=out)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = _lib.launch_count() - l0
    alg_bytes = 4.0 * n * (2 * m + 7)  # SURVEY s8d byte model
    peak, src = peaks()
    # e2e: host vectors in (pinned), host iterate out, every step
    hp = [(a.cpu().pin_memory(), b.cpu().pin_memory()) for a, b in stream[-args.steps:]]
    host_out = torch.empty(n, dtype=torch.float32).pin_memory()
    pd, gd = torch.empty_like(out), torch.empty_like(out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for a, b in hp:
        pd.copy_(a, non_blocking=True)
        gd.copy_(b, non_blocking=True)
        win.push(pd, gd)
        anderson.aa_step(win, weights=anderson.aa_weights(win), out=out)
        host_out.copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / len(hp)
    cpu = None
    if not args.no_cpu:
        import oracle
        nc = 5_000_000
        rng = np.random.default_rng(0)
        wo = oracle.AAWindowOracle(nc, m)
        vecs = [(rng.standard_normal(nc), rng.standard_normal(nc)) for _ in range(m + 3)]
        for k in range(m + 1):
            wo.push(*vecs[k])
        t0 = time.perf_counter()
        for k in range(m + 1, m + 3):
            wo.push(*vecs[k])
            oracle.aa_step(wo, 1.0, oracle.aa_weights(wo))
        cms = (time.perf_counter() - t0) * 1e3 / 2 * (n / nc)
        cpu = {"value": cms, "unit": "ms/iteration", "cores": os.cpu_count() or 1,
               "kind": "port", "sample": f"oracle AAWindow push+weights+step at N={nc}, m={m}, "
                                         "2 steady-state iterations, scaled x10 to N=5e7"}
    line = {"metric": "AA mixing step time (push + weights + step)", "value": ms,
            "unit": "ms/iteration", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 standalone AA mixing step: N=5e7 fp32, m=10, N(0,1) + "
                                   "rank-3 smooth component", "l2": "inputs larger than L2 "
                                   "(%.1f GB of window vectors)" % (2 * m * n * 4 / 1e9)},
            "e2e": {"value": e2e_ms, "unit": "ms/iteration", "h2d_bytes_per_step": 2 * n * 4,
                    "d2h_bytes_per_step": n * 4},
            "roofline": {"bound": "hbm", "kernel": "aa_push + aa_step",
                         "achieved": alg_bytes / (ms / 1e3) / 1e9, "peak": peak,
                         "peak_source": src, "unit": "GB/s",
                         "frac": alg_bytes / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "bytes_per_launch": alg_bytes},
            "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="weak: config shot count per rank (C3/C4 default); "
                         "strong: config shot count sharded over ranks (C1/C5 default)")
    args = ap.parse_args()
    if args.config == "c2":
        return run_c2(args) if args.impl != "reference" else run_reference_c2(args)
    if args.config == "c4" and args.impl != "reference":
        return run_lsrtm(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

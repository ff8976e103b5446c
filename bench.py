"""Benchmark: FWI gradient throughput of the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c1|c5|c2]
                    [--impl ours|reference]

Workload (default, BASELINE.json configs[2] = "C3"): one complete FWI gradient
per step -- 30 shots, 201x601 grid (241x641 padded), nt 4000, 8th-order
stencil, fp32, 20-cell sponge: forward sweep with history store, residual +
misfit, adjoint sweep with fused imaging, image reduction, fold, and (N > 1)
one all-reduce.  Shots are sharded over the N ranks in contiguous blocks
(SURVEY s8e): every config is its fixed BASELINE survey split over the ranks
(strong scaling: C3 30 -> 4,4,4,4,4,4,3,3 at N = 8, C5 240 -> 30 each);
--scaling weak gives every rank the config's full shot count instead.
Synthetic seeded layered-fault model (the paper's Marmousi is not available
offline).

The C3 line also carries ``c5_kernels``: the two boundary-saving step kernels
of C5 (band-storing forward, fused reverse-forward + adjoint) timed on the
full 1041 x 3041 padded grid over 14-shot launches (the batch a C5 gradient
runs) -- the HBM-bound case.

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


class NvmlClockSampler:
    """SM clocks + throttle reasons through NVML (nvidia_ml_py) every 20 ms
    during the timed region."""

    # nvmlClocksEventReason* bits
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
            "sw_power_cap": 0x4}

    def __init__(self, index):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                rs = fn(self.h)
                ut = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.rows.append((sm, mx, rs, ut))
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r[0] for r in self.rows if r[3] >= 50] or [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, b in self.BITS.items() if r[2] & b})
        counts = {k: sum(1 for r in self.rows if r[2] & b) for k, b in self.BITS.items()}
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml",
                "reason_samples": {k: v for k, v in counts.items() if v}}


def clock_sampler(index):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


def l2_cap_gbs(clocks):
    """L2 (LTS) throughput cap: ~6300 B/cycle full chip (measured,
    /opt/skills/guides/B300_MICROARCH.md) at the maximum SM clock.  Under the
    power cap the SM clock this run samples is lower, and the measured L2
    rate then exceeds 6300 B x that clock, so the L2 does not follow it."""
    mhz = (clocks or {}).get("sm_max_mhz")
    return 6300.0 * mhz * 1e6 / 1e9 if mhz else None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


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
    """Strong by default: the config's fixed survey (BASELINE.json) sharded
    over the ranks in contiguous blocks.  --scaling weak: every
    rank owns the config's shot count (a survey of shots * N)."""
    if args.scaling != "auto":
        return args.scaling
    return "strong"


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
    # every shot of the config when that stays a bounded sample (C3: all 30)
    shots = min(case["geometry"].n_sources, 2 * cores)
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
                             "cpu_model": cpu_model(), "sample": sample},
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
                                       "cpu_model": cpu_model(),
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
    with clock_sampler(local) as clk:
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
    # value counts the reference algorithm's stencil updates per LSRTM
    # gradient (BornKernel with every background cached,
    # seisopt/gradients.py:177-220): Born forward + adjoint = 2 sweeps per
    # shot.  Shots whose background is not cached here run extra sweeps
    # (lock-step background, and in CHECKPOINT / BOUNDARY mode its re-run in
    # the adjoint); those are reported as executed_gcell_per_s.
    nloc = kern._range()[1]
    cached = kern.cached
    recon = kern.ws.query()["recon"]
    per_uncached = 3 if recon == "full" else 4
    cells = 2.0 * S * nt * C
    executed = (2.0 * cached + per_uncached * (nloc - cached)) * nt * C * world
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
            "executed_gcell_per_s": executed * args.steps / (ms / 1e3) / 1e9,
            "sweeps_per_shot": {"cached": 2, "uncached": per_uncached},
            "e2e": {"value": cells * args.steps / e2e_s / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": p_host.nbytes, "d2h_bytes_per_step": p_host.nbytes + 8},
            "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": None}),
            flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def init_dist(dev, world):
    """NCCL process group (world > 1) with NCCL's init log on, so the
    communicator size each rank reports can be checked against WORLD_SIZE."""
    import torch.distributed as dist
    if world <= 1:
        return None
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist.init_process_group("nccl", device_id=dev)
    return dist


def shard_report(dist, world, shard, n_shots):
    """Every rank's (first shot, count) and the communicator size."""
    import torch
    s0, cnt = (shard.shot0, shard.count) if shard else (0, n_shots)
    if dist is None:
        return {"backend": None, "comm_nranks": 1, "shot_ranges": [[s0, cnt]]}
    t = torch.tensor([s0, cnt], dtype=torch.int64, device="cuda")
    allt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allt, t)
    return {"backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
            "shot_ranges": [[int(x[0]), int(x[1])] for x in allt]}


def c5_kernel_record(dev, peak, peak_src, reps=400, shots=14, nt=400):
    """BASELINE C5's boundary-saving step kernels on the full 1001 x 3001 grid
    (1041 x 3041 padded), `shots`-shot launches as the C5 gradient runs them
    (two concurrent chains): the band-storing forward and the fused
    reverse-forward + three-level adjoint with imaging, CUDA events over
    `reps` launches on the handle's stream.  nt only sizes the band store
    (the per-step work does not depend on it).  Algorithmic bytes per SURVEY
    s8d (stencil update 16 B, imaging 12 B per shot-cell); DRAM bytes from the
    committed ncu capture of the same kernels (profiles/traffic.json)."""
    from paper_2008_11778_b200 import synthetic
    from paper_2008_11778_b200.wavesim import Propagator
    case = synthetic.layered_case("c5", n_shots=shots, nt=nt)
    prop = Propagator(case["grid"], case["geometry"], case["wavelet"], case["config"],
                      dtype="float32", device=dev, recon="boundary")
    try:
        prop.set_model(case["init"].m)
        C = prop.shape[0] * prop.shape[1]
        es = 4
        ms_fwd = prop.time_step_kernel(6, shots, reps=reps)
        ms_adj = prop.time_step_kernel(5, shots, reps=reps)
    finally:
        prop.close()
    tr = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath)).get("c5", {})
    out = {"grid": "1041x3041 padded (C5)", "shots_per_launch": shots, "reps": reps,
           "peak": peak, "peak_source": peak_src}
    # kmin: the bytes the kernel as designed must move per shot-cell -- forward
    # u, inc in and out (16 B); fused reverse + adjoint with both three-level
    # recurrences: V_n, V_{n+1}, u_n, u_{n+1} in, V_{n-1}, u_{n-1} out (24 B;
    # the image read-modify-write adds 8 B per CTA group of up to 8 shots, the
    # band store is <6 % of cells)
    for name, ms, alg_b, kmin_b in (("forward_band_step", ms_fwd, 4 * es, 4 * es),
                                    ("reverse_adjoint_step", ms_adj, 8 * es + 3 * es, 6 * es)):
        alg = shots * C * alg_b
        dram = tr.get(name)
        dram_step = dram * shots if (dram is not None and tr.get("per_shot")) else dram
        out[name] = {
            "ms_per_step": ms, "alg_bytes_per_shot_cell": alg_b,
            "alg_gbs": alg / (ms / 1e3) / 1e9, "alg_frac": alg / (ms / 1e3) / 1e9 / peak,
            "kernel_min_bytes_per_shot_cell": kmin_b,
            "kernel_min_frac": shots * C * kmin_b / (ms / 1e3) / 1e9 / peak,
            "dram_bytes_per_step": dram_step,
            "dram_gbs": (dram_step / (ms / 1e3) / 1e9) if dram_step else None,
            "dram_frac": (dram_step / (ms / 1e3) / 1e9 / peak) if dram_step else None,
        }
    return out


def run_ours(args):
    import torch

    from paper_2008_11778_b200 import _lib, gradients, shards

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(dev, world)
    case = build_case(args.config, total_shots(args, world))
    geom, grid, cfg, wav = case["geometry"], case["grid"], case["config"], case["wavelet"]
    S, nt = geom.n_sources, geom.nt
    shard = shards.ShotShard.from_env(S) if world > 1 else None
    comm = shard_report(dist, world, shard, S)
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
    # the sweep buffers may take 80 % of what is free with the observed data
    # resident (C5: boundary-saving batches of 13 shots)
    budget = 0.0
    if args.config == "c5":
        torch.cuda.empty_cache()  # the synthesis temporaries go back to the driver first
        budget = 0.8 * torch.cuda.mem_get_info(dev)[0]
    obj = gradients.FwiObjective(grid, obs_full, wav, geom, cfg, dtype=case["dtype"],
                                 device=dev, shard=shard, mem_budget_bytes=budget)
    del obs_full
    torch.cuda.empty_cache()
    p_host = np.ascontiguousarray(case["init"].m.ravel())
    p_dev = torch.as_tensor(p_host, device=dev, dtype=obj.prop.tdtype)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        obj.value_and_grad(p_dev)
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    phases = {"forward": 0.0, "residual": 0.0, "adjoint": 0.0, "reduce": 0.0}
    with clock_sampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            val, grad = obj.value_and_grad(p_dev)
            # device time of this gradient's phases (events recorded on the
            # handle's stream, read after the call's own synchronisation)
            for k, v in obj.prop.phase_times().items():
                phases[k] += v
        e1.record(stream)
        barrier()
    launches = _lib.launch_count() - l0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
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
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    e2e_value = cells_per_grad * args.steps / e2e_s / 1e9
    nbytes = p_host.nbytes

    # Roofline of the dominant kernel.  Both step kernels launch nt times per
    # gradient; their live per-step time is the gradient's phase time / nt
    # (CUDA events on the launching stream around the captured sweep graphs,
    # a step = the whole batch as two concurrent half-batch chains), and the
    # dominant one is the phase with the larger share of the gradient.
    prop = obj.prop
    local_shots = shard.count if shard else S
    es = prop.esz
    q = prop.query()
    batches = -(-local_shots // min(local_shots, q["batch"]))
    # the library balances the batches (sizes differ by at most one): the
    # bytes of an average step are those of local_shots / batches shots
    launch_shots = local_shots / batches
    steps_run = args.steps * nt * batches
    ms_fwd = phases["forward"] / steps_run
    ms_adj = phases["adjoint"] / steps_run
    total_ph = sum(phases.values())
    if q["recon"] == "boundary":
        # band-storing forward (stencil 4s; the sponge-frame store is <6 % of
        # cells, not counted) and the fused reverse-forward + adjoint step
        # (two stencil updates 8s + imaging 3s)
        bytes_fwd = launch_shots * C * (4 * es)
        bytes_adj = launch_shots * C * (8 * es + 3 * es)
        names = ("forward_band_step", "reverse_adjoint_step")
        iso = (6, 5)
    else:
        bytes_fwd = launch_shots * C * (4 * es + es)       # stencil 4s + history store s
        bytes_adj = launch_shots * C * (4 * es + 3 * es)   # stencil 4s + imaging 3s
        names = ("forward_step", "adjoint_step")
        iso = (0, 1)
    if q["recon"] == "checkpoint":
        # the adjoint phase also re-runs the forward per segment
        bytes_adj += launch_shots * C * (4 * es + es)
    reps = 100 if launch_shots * C < 2e7 else 20
    iso_shots = -(-local_shots // batches)
    iso_fwd = prop.time_step_kernel(iso[0], iso_shots, reps=reps)
    iso_adj = prop.time_step_kernel(iso[1], iso_shots, reps=reps)
    peak, peak_src = peaks()
    kern = {}
    traffic_tab = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic_tab = json.load(open(tpath)).get(args.config, {})
        except Exception:
            traffic_tab = {}
    clocks = clk.summary()
    l2_cap = l2_cap_gbs(clocks)
    for name, msk, byt, ph, iso_ms in ((names[0], ms_fwd, bytes_fwd, phases["forward"], iso_fwd),
                                       (names[1], ms_adj, bytes_adj, phases["adjoint"], iso_adj)):
        tr = traffic_tab.get(name)
        lts = (traffic_tab.get("lts") or {}).get(name)
        if traffic_tab.get("per_shot"):
            tr = tr * launch_shots if tr is not None else None
            lts = lts * launch_shots if lts is not None else None
        elif args.config == "c3" and launch_shots != 30:
            # the committed C3 capture is of 30-shot steps
            tr = tr * launch_shots / 30.0 if tr is not None else None
            lts = lts * launch_shots / 30.0 if lts is not None else None
        kern[name] = {"ms_per_step": msk, "share": ph / total_ph if total_ph else None,
                      "bytes_per_step": byt, "achieved": byt / (msk / 1e3) / 1e9,
                      "frac": byt / (msk / 1e3) / 1e9 / peak, "traffic": tr,
                      "traffic_gbs": (tr / (msk / 1e3) / 1e9) if tr else None,
                      # L2 tag-stage bytes (ncu lts__t_bytes.sum, steady state) over
                      # the live step time, against the measured LTS cap of
                      # ~6300 B/cycle at the maximum SM clock
                      "l2_bytes_per_step": lts,
                      "l2_gbs": (lts / (msk / 1e3) / 1e9) if lts else None,
                      "l2_frac": (lts / (msk / 1e3) / 1e9 / l2_cap) if (lts and l2_cap) else None,
                      "isolated_ms_per_step": iso_ms}
    dom = max(names, key=lambda n: kern[n]["share"] or 0.0)
    dk = kern[dom]

    c5 = None
    if args.config == "c3" and rank == 0 and not args.no_c5_kernels:
        try:
            c5 = c5_kernel_record(dev, peak, peak_src)
        except Exception as exc:  # recorded, not fatal for the C3 line
            c5 = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        shots = min(S, cores)
        nts = {"c1": 800, "c3": 250, "c4": 150, "c5": 20}.get(args.config, 200)
        dt, cells = cpu_sample(case, cores, shots, nts)
        cpu = {"value": cells / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
               "cpu_model": cpu_model(),
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
            "comm": comm,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes + 8, "gradients_per_s": args.steps / e2e_s},
            "phases_ms_per_gradient": {k: v / args.steps for k, v in phases.items()},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dk["achieved"],
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": dk["frac"], "traffic": dk["traffic"],
                         # ncu DRAM bytes of the step / its live time: the HBM
                         # actually moved (C3 fields stay in L2, so < achieved)
                         "traffic_gbs": dk["traffic_gbs"],
                         "traffic_frac": (dk["traffic_gbs"] / peak) if dk["traffic_gbs"] else None,
                         "l2": {"gbs": dk["l2_gbs"], "cap_gbs": l2_cap, "frac": dk["l2_frac"],
                                "cap_source": "6300 B/cycle (B300_MICROARCH.md LTS cap) x "
                                              "max SM clock"},
                         "shots_per_step": launch_shots,
                         "chains": prop.chains(iso_shots),
                         "bytes_per_step": dk["bytes_per_step"], "ms_per_step": dk["ms_per_step"],
                         "share": dk["share"], "timing": "gradient phase events / steps",
                         "kernels": kern},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if c5 is not None:
            line["c5_kernels"] = c5
        print(json.dumps(line), flush=True)
    if dist is not None:
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
    recombination, window full and sliding.  On several GPUs N is sharded
    (SURVEY s8e): each rank's window holds N / world entries and the Gram row
    is summed over the ranks (one small all-reduce per push)."""
    import torch

    from paper_2008_11778_b200 import _lib, anderson, shards
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(dev, world)
    n_total, m = 50_000_000, 10
    n0, n = shards.shard_bounds(n_total, world, rank)
    total = m + 1 + args.warmup + args.steps
    stream = aa_stream_torch(n, total, rank, dev, torch.float32)
    win = anderson.AAWindow(n, m, dtype="float32", device=dev,
                            shard_group=True if dist is not None else None)
    out = torch.empty(n, device=dev, dtype=torch.float32)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for k in range(m + 1 + args.warmup):
        win.push(*stream[k])
        if win.m_k:
            anderson.aa_step(win, weights=anderson.aa_weights(win), out=out)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    with clock_sampler(local) as clk:
        barrier()
        e0.record()
        for k in range(m + 1 + args.warmup, total):
            win.push(*stream[k])
            w = anderson.aa_weights(win)
            anderson.aa_step(win, weights=w, out=out)
        e1.record()
        barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    launches = _lib.launch_count() - l0
    alg_bytes = 4.0 * n_total * (2 * m + 7)  # SURVEY s8d byte model, all ranks
    peak, src = peaks()
    # e2e: host vectors in (pinned), host iterate out, every step
    hp = [(a.cpu().pin_memory(), b.cpu().pin_memory()) for a, b in stream[-args.steps:]]
    host_out = torch.empty(n, dtype=torch.float32).pin_memory()
    pd, gd = torch.empty_like(out), torch.empty_like(out)
    barrier()
    t0 = time.perf_counter()
    for a, b in hp:
        pd.copy_(a, non_blocking=True)
        gd.copy_(b, non_blocking=True)
        win.push(pd, gd)
        anderson.aa_step(win, weights=anderson.aa_weights(win), out=out)
        host_out.copy_(out, non_blocking=True)
    barrier()
    te = torch.tensor([(time.perf_counter() - t0) * 1e3 / len(hp)], dtype=torch.float64,
                      device=dev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
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
        cms = (time.perf_counter() - t0) * 1e3 / 2 * (n_total / nc)
        cpu = {"value": cms, "unit": "ms/iteration", "cores": os.cpu_count() or 1,
               "cpu_model": cpu_model(),
               "kind": "port", "sample": f"oracle AAWindow push+weights+step at N={nc}, m={m}, "
                                         "2 steady-state iterations, scaled x10 to N=5e7"}
    if rank == 0:
        line = {"metric": "AA mixing step time (push + weights + step)", "value": ms,
                "unit": "ms/iteration", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "C2 standalone AA mixing step: N=5e7 fp32, m=10, N(0,1) + "
                                       "rank-3 smooth component", "n_per_rank": n,
                           "l2": "inputs larger than L2 (%.1f GB of window vectors per rank)"
                                 % (2 * m * n * 4 / 1e9)},
                "e2e": {"value": e2e_ms, "unit": "ms/iteration", "h2d_bytes_per_step": 2 * n * 4,
                        "d2h_bytes_per_step": n * 4},
                "roofline": {"bound": "hbm", "kernel": "aa_push + aa_step",
                             "achieved": alg_bytes / world / (ms / 1e3) / 1e9, "peak": peak,
                             "peak_source": src, "unit": "GB/s",
                             "frac": alg_bytes / world / (ms / 1e3) / 1e9 / peak, "traffic": None,
                             "bytes_per_launch": alg_bytes / world},
                "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5-kernels", action="store_true",
                    help="skip the C5 boundary-saving kernel record of the C3 line")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="strong (default): the config's survey sharded over the ranks; "
                         "weak: the config's shot count on every rank")
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

#!/usr/bin/env python
"""Benchmark of the hot path: one fused Vecchia loglik + gradient + Fisher-information
evaluation per step (BASELINE.json metric: observations / second at n = 2^20, m = 30).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (BASELINE.json configs[1]): n = 2^20 uniform points in [0,1]^2, p = 1, Matern 3/2
("matern15_isotropic"), theta = (1.0, 0.05, 0.1), m = 30, synthetic y ~ N(0,1), neighbor
table from the package's own host search.  BASELINE's metric fixes n = 2^20 for 1/2/4/8 GPUs, so
the default is STRONG scaling (`--scaling strong`: the 2^20 observations are split into N
contiguous row shards, dataset replicated); `--scaling weak` keeps 2^20 observations PER GPU.
One JSON line is printed by rank 0.

`value`     : obs/s with inputs resident in HBM; K steps timed with CUDA events, max over ranks.
`e2e`       : obs/s through the public API (engine.DeviceProblem from pinned HOST arrays ->
              evaluation -> totals on the host), H2D and D2H inside the timed region; MEAN step time
              (median and minimum beside it).
`roofline`  : the main kernel against the measured FP64 peak of this GPU = the better of the DFMA and
              the DMMA micro-kernel (both recorded).
`cpu_baseline` / `--impl reference`: the CPU implementation of the same path on the host
              cores (oracle port for Matern, which the reference lacks; the reference's own
              compiled core, oracle/_ref, is timed beside it on the exponential kernel).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "Vecchia loglik+grad+info evals: obs/sec at n=2^20, m=30"
UNIT = "obs/s"


def algorithmic_flops(family: str, d: int, p: int, q: int, m: int) -> dict:
    """flops per tail observation, every + - * / sqrt exp log = 1,
    FMA = 2, distance/exp once per pair.  F_min counts the variance/nugget shortcuts this
    kernel uses (c_0 = e_last/sigma^2, c_nugget = sigma^2 B^-1 u)."""
    k = m + 1
    T = k * (k - 1) // 2
    pair = {"exponential_isotropic": 3 * d + 6, "exponential_sphere": 3 * d + 6, "matern15_isotropic": 3 * d + 10,
            "matern25_isotropic": 3 * d + 13, "exponential_spacetime": 4 * d + 11,
            "exponential_anisotropic": 4 * d + 8 + 3 * d,
            # general Matern: 3 Bessel evaluations count as 1 "flop" each, like exp (SURVEY 8d convention)
            "matern_isotropic": 3 * d + 20}[family]
    qd = q - 2
    cov = T * pair + 2 * k
    chol = sum((a + 1) ** 2 for a in range(k))
    solves = (2 + p) * k * k
    dense = 4 * T + k + k * k
    contract = (2 + p + p * p) + q * (2 * k + 2 * k * p + 5 + 5 * p + 5 * p * p) + q * (q + 1) // 2 * (2 * k + 2)
    return {"F_generic": cov + chol + solves + q * dense + contract,
            "F_min": cov + chol + solves + qd * dense + (k + k * k) + contract}


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            self.nv = None

    def _loop(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "hw_power_brake_slowdown": 0x80, "sync_boost": 0x10, "applications_clocks_setting": 0x2}
        while not self._stop.is_set():
            try:
                self.samples.append(int(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                mask = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
                for name, bit in names.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._loop, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_workload(n_total: int, d: int, p: int, seed: int = 2407):
    rng = np.random.default_rng(seed)
    locs = rng.uniform(0.0, 1.0, (n_total, d))
    y = rng.normal(size=n_total)
    X = np.ones((n_total, p))
    for j in range(1, p):  # covariates: the coordinates, then their squares, ... (p - 1 may exceed d)
        X[:, j] = locs[:, (j - 1) % d] ** (1 + (j - 1) // d)
    return y, X, locs


def oracle_table(n, nn_rows, row0):
    """The C oracle indexes the neighbor table by global row: embed the shard rows (built ONCE per arm,
    outside every timed region -- a 260 MB fill at n = 2^20)."""
    full = np.full((n, nn_rows.shape[1]), -1, dtype=np.int64)
    full[row0:row0 + nn_rows.shape[0]] = nn_rows
    return full


def cpu_time_oracle(y, X, locs, full, row0, family, theta, rows, workers, repeats=1):
    """Best-of timing of the C oracle port over `rows` observations starting at row0; returns
    (seconds, totals of the last run)."""
    from oracle import vecchia_oracle as vo
    best, tot = float("inf"), None
    for _ in range(repeats):
        t0 = time.perf_counter()
        tot = vo.run(y, X, locs, full, family, theta, i0=row0, i1=row0 + rows, workers=workers, deterministic=False)
        best = min(best, time.perf_counter() - t0)
    return best, tot


def reference_arm(args):
    """--impl reference: the CPU implementation of the same evaluation on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import reference_core
    cores = os.cpu_count() or 1
    n_total = total_observations(args, args.gpus)
    y, X, locs = make_workload(n_total, args.d, args.p)
    theta = np.asarray(args.theta, dtype=np.float64)
    # bounded sample: rows from the middle of the workload, sized for ~ref_seconds of CPU work per step
    from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows
    probe = 1 << 14
    row0 = n_total // 2
    nn_probe = find_ordered_neighbor_rows(locs, args.m, row0, probe)
    t, _ = cpu_time_oracle(y, X, locs, oracle_table(n_total, nn_probe, row0), row0, args.family, theta, probe, cores)
    sample = int(min(n_total - row0, max(probe, (probe / t) * args.ref_seconds)))
    sample = 1 << int(np.floor(np.log2(sample)))
    nn_rows = find_ordered_neighbor_rows(locs, args.m, row0, sample)
    full = oracle_table(n_total, nn_rows, row0)  # once, outside the timed loop
    for _ in range(max(args.warmup, 2)):  # the first pass or two page in the 260 MB table and spin up the threads
        cpu_time_oracle(y, X, locs, full, row0, args.family, theta, sample, cores)
    each = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        each.append(cpu_time_oracle(y, X, locs, full, row0, args.family, theta, sample, cores)[0])
    sec = (time.perf_counter() - t0) / args.steps
    value = sample / sec
    kind = "port"
    extra = {}
    if reference_core.available() and n_total <= (1 << 21):
        # the reference's own compiled core has no Matern kernel: time it on the exponential
        # kernel over the same rows as context (same gather / Cholesky / solves, cheaper pair term)
        K = reference_core.module()
        q, pp = 3, args.p
        slots = (np.zeros(n_total), np.zeros(n_total), np.zeros((n_total, pp, pp)), np.zeros((n_total, pp)),
                 np.zeros((n_total, q)), np.zeros((n_total, q)), np.zeros((n_total, pp, q)),
                 np.zeros((n_total, pp, pp, q)), np.zeros((n_total, q, q)))
        failv = np.zeros(n_total, dtype=np.int32)
        th = np.array([theta[0], theta[1], theta[-1]])
        best = float("inf")
        for _ in range(2):
            t1 = time.perf_counter()
            K.RUNNERS["task"](y, X, locs, full, th, 0, 0.0, slots, failv, row0, row0 + sample, cores, 32)
            best = min(best, time.perf_counter() - t1)
        extra["reference_compiled_core_exp_iso_obs_per_s"] = sample / best
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": max(args.warmup, 2), "ms_per_step": 1000.0 * sec, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, n_total, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"rows [{row0}, {row0 + sample}) of the same workload per step "
                                   f"(C/OpenMP port of the reference kernel with the Matern 3/2 pair term; "
                                   f"the reference itself has no Matern family); neighbor table built once, "
                                   f"outside the timed loop", "ms_each": [round(1000.0 * t, 1) for t in each],
                         "best_step_obs_per_s": sample / min(each), **extra},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def total_observations(args, world):
    return args.n if args.scaling == "strong" else world * args.n


def workload_config(args, n_total, world, flush=None):
    per = -(-n_total // world)
    if flush is None:  # same rule as ours_arm: per-GPU inputs against 1.5 x the 126 MB L2
        flush = per * (args.m + 1) * 8 + n_total * 8 * (args.d + args.p + 1) < 1.5 * 126e6
    return {"workload": f"config2: n={n_total} total ({per} per GPU, {args.scaling} scaling), d={args.d}, p={args.p}, "
                        f"{args.family}, m={args.m}, theta={list(args.theta)}, one loglik+grad+info evaluation per step",
            "n_per_gpu": per, "n_total": n_total, "m": args.m, "family": args.family, "d": args.d, "p": args.p,
            "parallelism": f"observation shards x{world}, one all-reduce of L+1 doubles",
            "l2_policy": "L2 flushed between timed steps (a 256 MB device buffer is rewritten; steps timed one by one)"
                         if flush else "inputs larger than L2 (neighbor table %.0f MB + records %.0f MB per GPU streamed "
                                       "once per step)" % (per * (args.m + 1) * 8 / 1e6,
                                                           n_total * 8 * (args.d + args.p + 1) / 1e6)}


def ours_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2407_02740_b200 as vg
    from paper_2407_02740_b200 import _cabi, distributed, engine
    from paper_2407_02740_b200.preprocess import find_ordered_neighbor_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise vg.DeviceUnavailable("bench.py needs a CUDA device: the cuda core has no CPU fallback")
    # one rank per GPU; VB200_BENCH_BACKEND=gloo lets several ranks share one GPU (used only to
    # exercise the sharded code path on a single-GPU box -- never for reported numbers)
    backend = os.environ.get("VB200_BENCH_BACKEND", "nccl")
    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    n_total = total_observations(args, world)
    theta = np.asarray(args.theta, dtype=np.float64)
    q = theta.shape[0]
    y, X, locs = make_workload(n_total, args.d, args.p)
    i0, i1 = distributed.shard_bounds(n_total, world, rank)
    workers = max(1, (os.cpu_count() or 1) // world)
    t0 = time.perf_counter()
    nn_rows = find_ordered_neighbor_rows(locs, args.m, i0, i1 - i0, workers=workers)
    t_nn = time.perf_counter() - t0

    # pinned host copies (the e2e leg copies from these every step)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hy, hX, hl, hn = pin(y), pin(X), pin(locs), pin(nn_rows)
    ds = vg.Dataset(hy.numpy(), hX.numpy(), hl.numpy())
    table = vg.NeighborArray(hn.numpy())  # this rank's rows only

    def new_problem(family=args.family):
        return engine.DeviceProblem(ds, table, family, device=device, row0=i0, rows=i1 - i0, layout=args.layout,
                                     nn_is_shard=True)

    def step(prob, th=theta):
        if world == 1:
            # the single-GPU evaluation every fit iteration makes: vb200_eval = one launch, one pinned D2H of
            # L+2 doubles and the failure word, one stream synchronisation (all inside the C library)
            return prob.totals(th)
        vec = prob.totals_async(th)
        totals, first = distributed.combine_partials(vec)   # all-reduce + ONE pinned D2H of L+2 doubles
        if first >= 0:
            raise vg.NotPositiveDefinite(pivot=-1, observation=first)
        return totals

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # L2 policy: the per-GPU inputs (neighbor rows + point records) are streamed once per step; when they
    # do not exceed the 126 MB L2 comfortably (strong scaling at N >= 2) L2 is flushed between timed steps.
    in_bytes = (i1 - i0) * (args.m + 1) * 8 + n_total * 8 * (args.d + args.p + 1)
    flush = in_bytes < 1.5 * 126e6
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device) if flush else None

    prob = new_problem()
    prob.use_current_stream()
    prob.enable_timing(True)
    for _ in range(max(args.warmup, 3)):
        totals = step(prob)
    kernel_ms = []
    barrier()
    with ClockSampler(dev_index) as clocks:
        if not flush:
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            for _ in range(args.steps):
                totals = step(prob)
                kernel_ms.append(prob.last_kernel_ms())
            end.record()
            torch.cuda.synchronize()
            ms_total = start.elapsed_time(end)
        else:
            ms_total = 0.0
            for _ in range(args.steps):
                flush_buf.fill_(1)
                barrier()
                start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                start.record()
                totals = step(prob)
                end.record()
                torch.cuda.synchronize()
                ms_total += start.elapsed_time(end)
                kernel_ms.append(prob.last_kernel_ms())
    barrier()
    launches = args.steps * prob.last_launch_count
    kernel_name = prob.last_kernel_name
    layout_used = prob.layout_for(q)
    k_ms = float(np.mean(kernel_ms))
    rank_kernel_ms = [k_ms]
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t)
        gathered = [torch.zeros(1, dtype=torch.float64, device=device) for _ in range(world)]
        dist.all_gather(gathered, torch.tensor([k_ms], dtype=torch.float64, device=device))
        rank_kernel_ms = [float(g) for g in gathered]
    ms_per_step = ms_total / args.steps
    value = n_total / (ms_per_step * 1e-3)
    ev = vg.assemble(engine.parts_from_flat(totals, args.p, q), n_total)
    prob.close()

    # ---- the family BASELINE config 2 literally names: general-order Matern (Bessel K on the device) at
    #      smoothness 3/2, same rows, kernel time only ----
    extra = {}
    if rank == 0 and args.family == "matern15_isotropic" and not args.no_extras:
        try:
            thg = np.array([theta[0], theta[1], 1.5, theta[-1]])
            with new_problem("matern_isotropic") as pg:
                pg.enable_timing(True)
                pg.totals(thg)  # the first evaluation runs chunk by chunk behind the upload: not a kernel time
                gms = []
                for _ in range(2):
                    step_tot = pg.totals(thg)
                    gms.append(pg.last_kernel_ms())
                gq = 4
                gev = vg.assemble(engine.parts_from_flat(step_tot, args.p, gq), n_total) if world == 1 else None
                extra["matern_general_obs_per_s"] = (i1 - i0) / (min(gms) * 1e-3)
                extra["matern_general_kernel_ms"] = float(min(gms))
                extra["matern_general_kernel"] = pg.last_kernel_name
                if gev is not None:
                    extra["matern_general_loglik_minus_closed_form"] = gev.loglik - ev.loglik
        except Exception as err:  # noqa: BLE001 - an extra, never the headline
            extra["matern_general_error"] = str(err)[:200]

    # ---- end to end: pinned host arrays -> device -> evaluation -> host totals, every step ----
    e2e_steps = max(3, min(args.steps, 30))
    for _ in range(2):
        with new_problem() as pr:
            step(pr)
    barrier()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    es.record()
    e2e_each = []
    h2d_seen, narrowed = 0, False
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        with new_problem() as pr:
            step(pr)
            h2d_seen, narrowed = pr.h2d_bytes, pr.upload_narrowed
        e2e_each.append(1000.0 * (time.perf_counter() - t1))
    ee.record()
    torch.cuda.synchronize()
    barrier()
    # headline = MEAN step time (every step counts, outliers included); median and minimum beside it
    e2e_mean_ms = max(es.elapsed_time(ee), 1000.0 * (time.perf_counter() - t0)) / e2e_steps
    e2e_median_ms = float(np.median(e2e_each))
    if world > 1:
        t = torch.tensor([e2e_mean_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean_ms = float(t)
    # bytes copied per step, as counted by the constructor that copies them: y, X, locs as float64, the neighbor
    # table as int32 when the narrowed upload is on (int64 host rows narrowed by the host threads inside the timed
    # region, widened again on the device) -- the HOST input is the reference's int64 table either way
    h2d = int(h2d_seen)
    h2d_host_input = int(hy.numel() * 8 + hX.numel() * 8 + hl.numel() * 8 + hn.numel() * 8)
    d2h = int((engine.acc_len(args.p, q) + 2) * 8)

    # ---- roofline of the main kernel (FP64 bound; peak = best of the two FP64 micro-kernels, both recorded) ----
    ct = __import__("ctypes")
    dp = lambda a: a.ctypes.data_as(ct.POINTER(ct.c_double))
    b1, s1, b2, s2 = np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(1)
    lib = _cabi.load()
    _cabi.check(lib.vb200_measure_fp64_peak(dev_index, 0.4, dp(b1), dp(s1)), "fp64 peak (DFMA)")
    _cabi.check(lib.vb200_measure_fp64_peak_mma(dev_index, 0.4, dp(b2), dp(s2)), "fp64 peak (DMMA)")
    peak = max(float(s1[0]), float(s2[0]))
    F = algorithmic_flops(args.family, args.d, args.p, q, args.m)
    achieved = F["F_min"] * (i1 - i0) / (k_ms * 1e-3) * 1e-12
    traffic = None
    tfile = ROOT / "profiles" / "roofline_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get(kernel_name)
        except Exception:  # noqa: BLE001
            traffic = None
    # "bound": the path is FP64-vector bound, not HBM- or tensor-bound
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name, "layout": layout_used,
                "kernel_ms": k_ms, "kernel_share_of_step": k_ms / ms_per_step,
                "flops_per_obs": F["F_min"], "flops_per_obs_generic": F["F_generic"],
                "peak_dfma_tflops": {"burst": float(b1[0]), "sustained": float(s1[0])},
                "peak_dmma_tflops": {"burst": float(b2[0]), "sustained": float(s2[0])},
                "peak_source": "measured here, max(sustained DFMA micro-kernel, sustained DMMA m8n8k4 micro-kernel) "
                               "over 0.4 s each; MEASURED_PEAKS.json has no FP64 entry",
                "hbm_algorithmic_bytes_per_obs": 8 * (args.d + args.p + 1) + 8 * (args.m + 1),
                "hbm_frac_of_measured_peak": (8 * (args.d + args.p + 1) + 8 * (args.m + 1)) * (i1 - i0)
                                             / (k_ms * 1e-3) / 1e9 / _hbm_peak()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, n_total, world, flush),
        "clocks": clocks.summary(),
        "e2e": {"value": n_total / (e2e_mean_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_mean_ms, "ms_per_step_median": e2e_median_ms, "steps": e2e_steps,
                "ms_each": [round(x, 2) for x in e2e_each], "ms_min": round(float(min(e2e_each)), 3),
                "statistic": "mean over the timed steps (max of CUDA-event and host wall time)",
                "host_input_bytes_per_step": h2d_host_input, "table_narrowed_to_int32": bool(narrowed),
                "path": "engine.DeviceProblem(pinned host y/X/locs/nn): table " + ("narrowed to int32 by the host threads, " if narrowed else "")
                        + "uploaded in 16 chunks on a side stream" + (", widened on the device (vb200_widen_indices)" if narrowed else "")
                        + ", vb200_create + vb200_eval_async per chunk behind the copies -> totals on the host"},
        "gpu_launches": launches, "roofline": roofline,
        "loglik": ev.loglik, "neighbor_search_s": t_nn, "rank_kernel_ms": rank_kernel_ms,
        "step_minus_kernel_us": 1000.0 * (ms_per_step - max(rank_kernel_ms)),
    }
    if extra:
        line["extra"] = extra
    if world > 1 and backend == "nccl":
        line["nccl"] = {"version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                        "NCCL_DEBUG": os.environ.get("NCCL_DEBUG", "")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, ds, table, y, X, locs, nn_rows, theta, device)
    if rank == 0 and world == 1 and not args.no_extras:
        line.setdefault("extra", {})["config1_fit"] = config1_fit_times()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6650.0  # the profiling guide's fallback


def cpu_baseline(args, ds, table, y, X, locs, nn_rows, theta, device):
    """The oracle port timed on the host cores over a bounded sample (about 10-20 s of CPU work), and a
    parity check of the GPU totals against the oracle's on exactly those rows at the bench theta."""
    from oracle import reference_core
    from paper_2407_02740_b200 import engine
    cores = os.cpu_count() or 1
    n = y.shape[0]
    probe = 1 << 14
    row0 = n // 2
    full = oracle_table(n, nn_rows, 0)  # once, outside the timers
    t, _ = cpu_time_oracle(y, X, locs, full, row0, args.family, theta, probe, cores)
    sample = int(min(n - row0, max(probe, (probe / t) * 8.0)))
    sample = 1 << int(np.floor(np.log2(sample)))
    best, cpu_tot = cpu_time_oracle(y, X, locs, full, row0, args.family, theta, sample, cores, repeats=2)
    out = {"value": sample / best, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"rows [{row0}, {row0 + sample}) of the same workload, best of 2 "
                     f"(C/OpenMP port with the Matern 3/2 pair term; the reference has no Matern family)"}
    # parity on the sampled rows: GPU totals over [row0, row0+sample) against the oracle's, entry by entry,
    # relative to max(|entry|, 1e-9 of the largest entry)
    with engine.DeviceProblem(ds, table, args.family, device=device, layout=args.layout, upload_chunks=1) as prob:
        gpu_tot = prob.totals(theta, i0=row0, i1=row0 + sample)
    scale = np.maximum(np.abs(cpu_tot), 1e-9 * np.abs(cpu_tot).max())
    out["parity_check"] = {"max_rel": float(np.max(np.abs(gpu_tot - cpu_tot) / scale)), "rows": int(sample),
                           "theta": [float(v) for v in theta],
                           "what": "GPU totals vs the CPU oracle's over the sampled rows, all L accumulator entries"}
    if reference_core.available() and n <= (1 << 21):
        K = reference_core.module()
        pp, q = args.p, 3
        slots = (np.zeros(n), np.zeros(n), np.zeros((n, pp, pp)), np.zeros((n, pp)), np.zeros((n, q)), np.zeros((n, q)),
                 np.zeros((n, pp, q)), np.zeros((n, pp, pp, q)), np.zeros((n, q, q)))
        failv = np.zeros(n, dtype=np.int32)
        th = np.array([theta[0], theta[1], theta[-1]])
        bt = float("inf")
        for _ in range(2):
            t1 = time.perf_counter()
            K.RUNNERS["task"](y, X, locs, full, th, 0, 0.0, slots, failv, row0, row0 + sample, cores, 32)
            bt = min(bt, time.perf_counter() - t1)
        out["reference_compiled_core_exp_iso_obs_per_s"] = sample / bt
        out["reference_note"] = ("oracle/_ref = the reference's own compiled core (run_task), exponential_isotropic "
                                 "kernel on the same rows")
    return out


_CONFIG1_CHILD = r"""
import json, sys, time
t0 = time.perf_counter()
sys.path.insert(0, %(root)r)
import numpy as np
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import inference, preprocess, simulate
t_import = time.perf_counter() - t0
mode, path = sys.argv[1], sys.argv[2]
n, m = 10000, 30
if mode == "gen":    # data for the fit: a draw from the model itself (device simulation), saved for the timing run
    rng = np.random.default_rng(11)
    locs = rng.uniform(size=(n, 2))
    locs = locs[preprocess.maxmin_ordering(locs).perm]
    X = np.ones((n, 1))
    nn = preprocess.find_ordered_neighbors(locs, m)
    truth = vg.CovarianceParameters("exponential_isotropic", np.array([2.0, 0.1, 0.1]))
    y = simulate.simulate_nn_gp(truth, np.array([1.0]), locs, X, nn, seed=5)
    np.savez(path, y=y, X=X, locs=locs, nn=nn.idx)
    sys.exit(0)
z = np.load(path)
ds = vg.Dataset(z["y"], z["X"], z["locs"])
nn = vg.NeighborArray(z["nn"])
model = vg.ModelSpec(covariance=inference.default_start(ds, "exponential_isotropic"), m=m, ordering="maxmin")
times = []
for _ in range(2):   # the FIRST fit is the first thing this process does on the GPU
    t1 = time.perf_counter()
    res = inference.fit(ds, nn, model)
    times.append(time.perf_counter() - t1)
print("RESULT " + json.dumps({"import_s": t_import, "fit_cold_s": times[0], "fit_warm_s": times[1],
                              "iterations": int(res.iterations), "evaluate_ms_warm": res.phase_timings["evaluate_ms"],
                              "theta_hat": [float(v) for v in res.theta_hat.theta], "n": n, "m": m}))
"""


def config1_fit_times():
    """BASELINE config 1 (n = 10^4, exponential_isotropic, m = 30, maxmin ordering, full Fisher-scoring fit) in a
    FRESH process: `fit_cold_s` is the first fit, which is also the process's first GPU work (CUDA context,
    library and kernel-module load, first upload included), `fit_warm_s` the second."""
    import subprocess, tempfile
    try:
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "config1.npz")
            code = _CONFIG1_CHILD % {"root": str(ROOT)}
            subprocess.run([sys.executable, "-c", code, "gen", path], capture_output=True, text=True, timeout=300, check=True)
            r = subprocess.run([sys.executable, "-c", code, "fit", path], capture_output=True, text=True, timeout=300)
        for ln in r.stdout.splitlines():
            if ln.startswith("RESULT "):
                return json.loads(ln[7:])
        return {"error": (r.stderr or r.stdout)[-300:]}
    except Exception as err:  # noqa: BLE001
        return {"error": str(err)[:300]}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", "--n-per-gpu", dest="n", type=int, default=1 << 20,
                    help="observations: in total (--scaling strong, the default) or per GPU (--scaling weak)")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong: n fixed at every GPU count, as BASELINE's metric reads; weak: n per GPU fixed")
    ap.add_argument("--no-extras", action="store_true", help="skip the general-Matern and config-1 extras")
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--p", type=int, default=1)
    ap.add_argument("--family", default="matern15_isotropic")
    ap.add_argument("--theta", type=float, nargs="+", default=[1.0, 0.05, 0.1])
    ap.add_argument("--layout", default="auto", choices=("auto", "warp_smem", "tiled_reg", "thread_smem", "thread_local"))
    ap.add_argument("--ref-seconds", type=float, default=2.0, help="target CPU seconds per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return reference_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())

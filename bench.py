#!/usr/bin/env python3
"""QAOA MaxCut energy on B200: lightcones/s for 3-regular N=30 p=4 (BASELINE.json).

One "step" = one full energy evaluation: all 45 edge lightcones of
random_regular(30, 3, 104478) at the acceptance-scale angles
(proj/tests/acceptance.cpp:70-71), contracted by bucket elimination.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value : device-resident throughput -- the plan (schedules, descriptors) and the
        gate table are in HBM; K executions of the level-batched program (CUDA
        graph: level kernels + fused-chain segment kernels) timed with CUDA
        events on the library's stream, L2 flushed between steps (the 512 MiB
        flush is outside the timed region), max over ranks.
e2e   : the public API end to end -- energy_expectation(graph, angles) with host
        inputs: host schedule construction, H2D of descriptors + gate table,
        kernels, D2H of the per-edge terms (+ the NCCL reduce for N>1),
        wall-clock, max over ranks.  The one-shot call pipelines lightcone
        chunks over 3 stream lanes (chunk c+1 is planned on the host while
        chunks <= c run), so host planning overlaps device work.
Multi-GPU: edges LPT-sharded by predicted work (the library's qtng_shard_edges,
the placement its single-process driver qtng_energy_multi uses too), one NCCL
reduce of the terms (total work fixed as N grows: "strong" scaling).
Sub-records (N=1, rank 0): `c4` (N=100 p=3, the 8-GPU config, on one GPU:
value, e2e, parity), `c64` (C2 in the complex64 mode: value, error),
`multi_api` (qtng_energy_multi on this one device: the C-ABI multi-GPU path)
and `merged` (C2 with merge_buckets: value, e2e, parity).
--impl reference: the reference's own energy_expectation (oracle/_ref, built
from /root/reference unmodified), matmul backend, jobs = all host threads.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C2": dict(n=30, d=3, seed=104478, gammas=[0.30, 0.25, 0.20, 0.15],
               betas=[0.35, 0.30, 0.25, 0.20],
               workload="QAOA MaxCut energy, random 3-regular N=30 p=4, seed 104478, 45 lightcones"),
    "C4": dict(n=100, d=3, seed=1, gammas=[0.30, 0.25, 0.20], betas=[0.35, 0.30, 0.25],
               workload="QAOA MaxCut energy, random 3-regular N=100 p=3, seed 1, 150 lightcones"),
}
METRIC = "QAOA MaxCut energy wall-time & lightcones/s (3-reg N=30 p=4) at 1/2/4/8 B200"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic(*kernels):
    """DRAM read+write bytes per step of `kernels` (summed), from the newest
    committed ncu launch list (profiles/<tag>/traffic.json, written by
    tools/summarize_profiles.py; tags sort by round and letter) -- ncu numbers
    are never measured here."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")))
    for fn in reversed(files):
        with open(fn) as f:
            t = json.load(f)
        per = t.get("dram_bytes_per_step", {})
        if kernels[0] in per:
            return {"traffic": sum(per.get(k, 0.0) for k in kernels), "traffic_source": t["source"]}
    return {"traffic": None}


def fp64_pipe_peak(dev_index, sm_max_mhz, lanes=64):
    """FP64 pipe issue peak in op/s: SMs x 64 FP64 lanes x SM clock.  The
    bucket loop is DMUL/DADD (one op per lane per clock each); NVIDIA's 37
    TFLOP/s figure counts a DFMA as two.  lanes=128: the FP32 pipe (c64 mode)."""
    import torch
    sms = torch.cuda.get_device_properties(dev_index).multi_processor_count
    return sms * lanes * (sm_max_mhz or 1965.0) * 1e6, sms


def measured_fp64_peak(q, dev_index):
    """The FP64 rates measured on this GPU right now by the library's own
    microkernels (qtng_fp64_peak, csrc/peak.cu): DMUL+DADD op/s, DFMA flop/s."""
    try:
        return q.fp64_peak(dev_index)
    except Exception:
        return None, None


def golden_energy(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "energies.json")) as f:
            return json.load(f)["configs"][name]["energy_naive"]
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML,
    else nvidia-smi)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        # seconds between NVML samples; bench.py lengthens it for the e2e phase,
        # whose host planning shares the CPU (and the driver) with the sampler
        self.interval = 0.005
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        # in-process NVML queries (~0.1 ms each): many samples even inside a
        # timed region of a few tens of milliseconds
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = get_reasons(h)
                self.samples.append([str(sm), str(mx), hex(r)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(self.interval)
        finally:
            pynvml.nvmlShutdown()

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np  # noqa: F401
    import oracle as O

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libqtnsim_ref.so missing (build needs /root/reference)"}))
        return 0
    jobs = cpu_threads()
    edges = O.ref_random_regular(cfg["n"], cfg["d"], cfg["seed"])
    m = len(edges)
    # One warm-up to size the sample: full energies when K of them fit in
    # ~150 s, otherwise a rotating subset of edges per step (same metric).
    t0 = time.perf_counter()
    e_full, _, _, _ = O.ref_energy(cfg["n"], edges, cfg["gammas"], cfg["betas"], "matmul",
                                   jobs=jobs)
    t_full = time.perf_counter() - t0
    per_step = m
    if t_full * args.steps > 150.0:
        per_step = max(jobs, int(m * 150.0 / (t_full * args.steps)))
        per_step = min(per_step, m)
    times, done = [], 0
    for step in range(max(0, args.warmup - 1) + args.steps):
        t0 = time.perf_counter()
        if per_step == m:
            O.ref_energy(cfg["n"], edges, cfg["gammas"], cfg["betas"], "matmul", jobs=jobs)
        else:
            sel = [(step * per_step + i) % m for i in range(per_step)]
            O.ref_edge_terms(cfg["n"], edges, cfg["gammas"], cfg["betas"], "matmul", jobs=jobs,
                             select=sel)
        dt = time.perf_counter() - t0
        if step >= max(0, args.warmup - 1):
            times.append(dt)
            done += per_step
    total = sum(times)
    value = done / total
    sample = (f"{'full energy' if per_step == m else f'{per_step} of {m} lightcones'} per step, "
              f"matmul backend, jobs={jobs}, OPENBLAS_NUM_THREADS=1")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "lightcones/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded random 3-regular graph)",
        "config": {"workload": cfg["workload"], "backend": "matmul", "jobs": jobs},
        "energy": e_full,
        "cpu_baseline": {"value": value, "unit": "lightcones/s", "cores": jobs, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "lightcones/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ B200 arm
def run_b200(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2204_06045_b200 as q
    from paper_2204_06045_b200 import dist as qd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = q.Context(local)
    g = q.random_regular(cfg["n"], cfg["d"], cfg["seed"])
    a = q.Angles(cfg["gammas"], cfg["betas"])
    p = a.depth()
    shards = qd.shards_for(q, g, p, world)
    mine = shards[rank]
    ecfg = q.EngineConfig(dtype=args.dtype)
    plan = q.Plan(g, p, edges=mine, ctx=ctx, cfg=ecfg)
    info = plan.info()

    def energy_step_device():
        return plan.execute(a)

    # warm-up (also the parity check)
    for _ in range(max(1, args.warmup)):
        terms = energy_step_device()
        plan.run_device(1)
    plan.profile(a)  # eager run with per-level / per-kernel events
    full = qd.scatter_terms(g.m, mine, terms)
    if world > 1:
        full = qd.reduce_terms(full, dev)
    energy = qd.energy_from_terms(g.m, full) if rank == 0 else None
    level_ms = plan.level_ms()
    lvl_kernel_ms = float(np.sum(level_ms))
    kms = plan.kernel_ms()

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clocks = ClockSampler(local)
    # ---- value: device-resident, L2 flushed between steps
    barrier()
    launches0 = q.kernel_launches()
    with clocks:
        total_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            total_ms += plan.run_device(1)
        barrier()
        # ---- e2e: public API with host inputs
        clocks.interval = float(os.environ.get("QTNG_BENCH_E2E_SAMPLE_S", "0.005"))
        l_value = q.kernel_launches() - launches0
        for _ in range(max(3, args.warmup)):
            q.energy_expectation(g, a, q.GpuBackend(ctx), edges=mine, cfg=ecfg)
        barrier()
        l_e2e0 = q.kernel_launches()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = q.energy_expectation(g, a, q.GpuBackend(ctx), edges=mine, cfg=ecfg)
            if world > 1:
                qd.reduce_terms(qd.scatter_terms(g.m, mine, res.terms), dev)
        barrier()
        e2e_s = time.perf_counter() - t0
        l_e2e = q.kernel_launches() - l_e2e0
        # ---- e2e with the angle-independent plan cached (QAOA optimiser loop):
        # H2D gate table, kernels, D2H terms per step
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            t = plan.execute(a)
            if world > 1:
                qd.reduce_terms(qd.scatter_terms(g.m, mine, t), dev)
        barrier()
        warm_s = time.perf_counter() - t0
    launches = {"value": l_value, "e2e": l_e2e}
    total_ms = max_over_ranks(total_ms)
    e2e_s = max_over_ranks(e2e_s)
    warm_s = max_over_ranks(warm_s)
    lvl_kernel_ms = max_over_ranks(lvl_kernel_ms)
    kms = {k: max_over_ranks(v) for k, v in kms.items()}

    # largest-bucket level in isolation (C3-class microbench on real buckets)
    big_level, big_bytes, big_ms = plan.time_level(-1, 20)
    # BASELINE configs[2]: the calibration bucket [w,2]->w-1 (engine.cpp:371-390)
    # as one level_kernel op, HBM-bound, timed alone (rank 0 only)
    c3 = microbench_c3(ctx) if rank == 0 and not args.no_c3 else None
    subs = {}
    if world == 1 and not args.no_sub:
        subs["c4"] = sub_c4(q, ctx, args)
        if args.dtype == "c128":
            subs["c64"] = sub_c64(q, ctx, cfg, args)
        subs["multi_api"] = sub_multi(q, ctx, cfg, args)
        if args.dtype == "c128":
            subs["merged"] = sub_merged(q, ctx, cfg, args)
    mpk_ma, mpk_fma = measured_fp64_peak(q, local)

    if rank != 0:
        return 0
    peak, peak_kind = load_peaks()
    ms_per_step = total_ms / args.steps
    value = g.m * args.steps / (total_ms / 1e3)
    gold = golden_energy(args.config)
    csum = clocks.summary()
    c64 = args.dtype == "c64"
    fp_peak_derived, sms = fp64_pipe_peak(local, csum.get("sm_max_mhz"), 128 if c64 else 64)
    fp_peak = mpk_ma if (mpk_ma and not c64) else fp_peak_derived
    # per-kernel device time INSIDE the measured graph replay: the step time
    # apportioned by the kernels' shares of the eager run's per-kernel CUDA
    # events (the kernels of one level overlap, so these shares sum the
    # kernels' own durations; the result never exceeds ms_per_step)
    ksum = max(1e-9, sum(kms.values()))
    kshare = {k: v / ksum for k, v in kms.items()}
    seg_share = kshare["seg_kernel"] + kshare.get("seg4_kernel", 0.0)  # the fused-chain kernels
    seg_s = ms_per_step * seg_share / 1e3
    lvl_s = ms_per_step * kshare["level_kernel"] / 1e3
    seg_ach = info.seg_fp64_ops / seg_s / 1e12 if seg_s > 0 else None
    lvl_ach = info.single_alg_bytes / lvl_s / 1e9 if lvl_s > 0 else None
    out = {
        "metric": METRIC, "value": value, "unit": "lightcones/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (seeded random 3-regular graph, acceptance-scale angles)",
        "config": {"workload": cfg["workload"], "parallelism": f"lightcone-sharded x{world}",
                   "l2": "512 MiB flush between timed steps (outside the timed region)",
                   "buckets": int(info.n_buckets), "levels": int(info.n_levels),
                   "max_width": int(info.max_width)},
        "energy": energy, "energy_golden_naive": gold,
        "parity_bit_exact": (energy == gold) if gold is not None and args.dtype == "c128" else None,
        "parity_rel_err": (abs(energy - gold) / abs(gold)) if gold else None,
        "e2e": {"value": g.m * args.steps / e2e_s, "unit": "lightcones/s",
                "h2d_bytes_per_step": int(info.desc_bytes + 16 * (2 + 4 * p) * 4),
                "d2h_bytes_per_step": int(16 * len(mine)),
                "ms_per_step": 1e3 * e2e_s / args.steps,
                "includes": "host schedule build (all edges, host threads, pipelined with the "
                            "device over 3 lanes) + H2D + kernels + D2H"},
        "e2e_plan_cached": {"value": g.m * args.steps / warm_s, "unit": "lightcones/s",
                            "h2d_bytes_per_step": int(16 * (2 + 4 * p) * 4),
                            "d2h_bytes_per_step": int(16 * len(mine)),
                            "ms_per_step": 1e3 * warm_s / args.steps,
                            "includes": "Plan.execute(angles): H2D gate table + kernels + D2H "
                                        "(schedules/descriptors built once per graph)"},
        # dominant kernel: the fused-chain seg_kernel keeps every chain
        # intermediate in registers, so it is bound by the FP64 pipe, not HBM
        "roofline": {"bound": "fp32" if c64 else "fp64",
                     "kernel": "seg_kernel + seg4_kernel (fused chains, all levels)",
                     "achieved": seg_ach, "peak": fp_peak / 1e12, "unit": "TFLOP/s",
                     "frac": (seg_ach * 1e12 / fp_peak) if seg_ach else None,
                     "peak_source": (f"derived: {sms} SMs x 128 FP32 lanes x sm_max_mhz" if c64 else
                                     ("measured in this run: qtng_fp64_peak (csrc/peak.cu), "
                                      "DMUL+DADD ops/s over 8 independent chains per thread"
                                      if mpk_ma else
                                      f"derived: {sms} SMs x 64 FP64 lanes x sm_max_mhz")),
                     "peak_derived": fp_peak_derived / 1e12,
                     "peak_fma_tflops_measured": (mpk_fma / 1e12) if mpk_fma else None,
                     **committed_traffic("seg_kernel", "seg4_kernel"),
                     "flops_per_step": info.seg_fp64_ops,
                     "flops_def": "the reference NaiveBackend loop's FP64 mul+add count of the "
                                  "buckets the fused-chain kernels evaluate",
                     "kernel_ms_per_step": ms_per_step * seg_share,
                     "kernel_ms_def": "ms_per_step (graph replay) x the fused-chain kernels' share "
                                      "of the per-kernel event times of an eager run",
                     "eager_kernel_ms": kms,
                     "share_of_kernel_time": seg_share},
        "roofline_level_kernel": {"bound": "hbm", "kernel": "level_kernel (unfused buckets)",
                                  "achieved": lvl_ach, "peak": peak, "unit": "GB/s",
                                  "frac": (lvl_ach / peak) if lvl_ach else None,
                                  "peak_source": peak_kind,
                                  **committed_traffic("level_kernel"),
                                  "alg_bytes_per_step": info.single_alg_bytes,
                                  "kernel_ms_per_step": ms_per_step * kshare["level_kernel"]},
        "roofline_step": {"alg_bytes_per_step": info.alg_bytes,
                          "dev_bytes_per_step": info.dev_bytes,
                          "fp64_ops_per_step": info.fp64_ops,
                          "effective_GBps": info.alg_bytes / (ms_per_step / 1e3) / 1e9,
                          "unfused_hbm_roofline_ms": info.alg_bytes / (peak * 1e9) * 1e3,
                          "fp64_roofline_ms": info.fp64_ops / fp_peak * 1e3,
                          "fused_hbm_floor_ms": info.dev_bytes / (peak * 1e9) * 1e3,
                          "fused_floors_note": "the fused program's own floors: dev_bytes at "
                                               "measured HBM, fp64_ops at the FP64 peak above",
                          "level_events_ms": lvl_kernel_ms,
                          "note": "alg_bytes = the reference's per-bucket accounting "
                                  "(SURVEY 8a); dev_bytes = what the fused program must move"},
        "roofline_largest_level": {"level": big_level, "alg_bytes": big_bytes, "ms": big_ms,
                                   "effective_GBps": big_bytes / (big_ms / 1e3) / 1e9},
        "microbench_c3": c3,
        "clocks": csum,
        "gpu_launches": int(launches["value"] + launches["e2e"]),
        "gpu_launches_detail": {**launches,
                                "note": "counted by the library (qtng_kernel_launches) inside the "
                                        "timed regions: value = graph replays, e2e = the pipelined "
                                        "one-shot calls"},
        "arena_bytes": int(info.arena_bytes),
        "segments": int(info.n_segments), "fused_buckets": int(info.n_fused_ops),
    }
    out.update(subs)
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def _golden_config(name):
    with open(os.path.join(ROOT, "tests", "golden", "energies.json")) as f:
        return json.load(f)["configs"][name]


def sub_c4(q, ctx, args, steps=10):
    """BASELINE configs[3] (N=100 p=3, the 8-GPU config) on this one GPU:
    device-resident value (graph replay), e2e through energy_expectation,
    parity against the reference's naive energy, and the LPT shard balance
    the 8-way run would see (predicted work)."""
    import numpy as np
    import torch
    from paper_2204_06045_b200 import dist as qd
    cfg = CONFIGS["C4"]
    g = q.random_regular(cfg["n"], 3, cfg["seed"])
    a = q.Angles(cfg["gammas"], cfg["betas"])
    plan = q.Plan(g, 3, ctx=ctx)
    terms = plan.execute(a)
    plan.run_device(3)
    dev_ms = plan.run_device(steps) / steps
    replay_terms = plan.terms()
    acc = 0.0  # engine.cpp:549-551: sum in edge order, then m/2 - sum/2
    for x in replay_terms.real:
        acc += float(x)
    e = 0.5 * g.m - 0.5 * acc
    for _ in range(2):
        q.energy_expectation(g, a, q.GpuBackend(ctx))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = q.energy_expectation(g, a, q.GpuBackend(ctx))
    e2e_ms = 1e3 * (time.perf_counter() - t0) / steps
    gold = _golden_config("C4")
    work = q.edge_work(g, 3)
    shards = qd.shards_for(q, g, 3, 8)
    loads = [float(sum(work[i] for i in s)) for s in shards]
    info = plan.info()
    plan.close()
    return {"workload": cfg["workload"], "value": g.m / (dev_ms / 1e3), "unit": "lightcones/s",
            "ms_per_step": dev_ms, "e2e": {"value": g.m / (e2e_ms / 1e3), "ms_per_step": e2e_ms},
            "energy": res.energy, "energy_golden_naive": gold["energy_naive"],
            "parity_bit_exact": res.energy == gold["energy_naive"] and
            bool(np.array_equal(replay_terms, terms)) and e == res.energy,
            "levels": int(info.n_levels), "buckets": int(info.n_buckets),
            "lpt8_predicted_speedup": float(sum(loads) / max(loads)),
            "note": "seed 1 (the golden config); its largest lightcone caps 8-way lightcone "
                    "sharding (SURVEY 8e)"}


def sub_c64(q, ctx, cfg, args, steps=10):
    """The complex64 mode (north_star: 1e-5) on the headline C2 workload."""
    g = q.random_regular(cfg["n"], cfg["d"], cfg["seed"])
    a = q.Angles(cfg["gammas"], cfg["betas"])
    plan = q.Plan(g, a.depth(), ctx=ctx, cfg=q.EngineConfig(dtype="c64"))
    plan.execute(a)
    plan.run_device(3)
    dev_ms = plan.run_device(steps) / steps
    t = plan.terms()
    acc = 0.0
    for x in t.real:
        acc += float(x)
    e = 0.5 * g.m - 0.5 * acc
    gold = golden_energy("C2")
    plan.close()
    return {"value": g.m / (dev_ms / 1e3), "unit": "lightcones/s", "ms_per_step": dev_ms,
            "dtype": "c64", "energy": e, "rel_err_vs_c128_golden": abs(e - gold) / abs(gold),
            "tolerance": 1e-5}


def sub_merged(q, ctx, cfg, args, steps=10):
    """C2 with merge_buckets (engine.cpp:306-358): merged buckets sum up to 9
    vars at once and run in the level kernel's multi-sum path; device value,
    one-shot e2e and parity against the reference's naive merged energy."""
    import numpy as np
    g = q.random_regular(cfg["n"], cfg["d"], cfg["seed"])
    a = q.Angles(cfg["gammas"], cfg["betas"])
    plan = q.Plan(g, a.depth(), merged=True, ctx=ctx)
    plan.execute(a)
    plan.run_device(3)
    dev_ms = plan.run_device(steps) / steps
    t = plan.terms()
    plan.profile(a)
    kms = plan.kernel_ms()
    info = plan.info()
    plan.close()
    t0 = time.perf_counter()
    for _ in range(3):
        res = q.energy_expectation(g, a, q.GpuBackend(ctx), merged=True)
    e2e_ms = 1e3 * (time.perf_counter() - t0) / 3
    try:
        with open(os.path.join(ROOT, "tests", "golden", "merged.json")) as f:
            gold = json.load(f)["C2"]
        ref = np.array([complex(x, y) for x, y in gold["terms_naive"]])
        exact = bool(np.array_equal(t, ref)) and res.energy == gold["energy_naive"]
        e_gold = gold["energy_naive"]
    except Exception:
        exact, e_gold = None, None
    return {"value": g.m / (dev_ms / 1e3), "unit": "lightcones/s", "ms_per_step": dev_ms,
            "e2e_ms_per_step": e2e_ms, "energy": res.energy, "energy_golden_naive_merged": e_gold,
            "parity_bit_exact": exact, "merges_applied": res.report.merges_applied,
            "eager_kernel_ms": kms, "levels": int(info.n_levels), "buckets": int(info.n_buckets),
            "dev_bytes": info.dev_bytes, "fp64_ops": info.fp64_ops}


def sub_multi(q, ctx, cfg, args, steps=5):
    """qtng_energy_multi (the single-process multi-GPU C driver: LPT shards,
    one host thread per device, one ncclReduce) on the one device here."""
    g = q.random_regular(cfg["n"], cfg["d"], cfg["seed"])
    a = q.Angles(cfg["gammas"], cfg["betas"])
    try:
        res, ms = q.energy_multi(g, a, [ctx])
        t0 = time.perf_counter()
        for _ in range(steps):
            res, ms = q.energy_multi(g, a, [ctx])
        wall = 1e3 * (time.perf_counter() - t0) / steps
    except Exception as ex:  # reported, not fatal
        return {"error": repr(ex)}
    return {"devices": 1, "e2e_ms_per_step": wall, "shard_ms": [float(x) for x in ms],
            "energy": res.energy, "parity_bit_exact": res.energy == golden_energy("C2")}


def microbench_c3(ctx, widths=(26, 28)):
    """The single-bucket microbench (BASELINE configs[2]): calibrate()'s
    synthetic bucket, a rank-w tensor times a rank-2 one summing the MSB var
    ([w, 2] -> w-1, 16*(2^w + 4 + 2^(w-1)) algorithmic bytes), contracted by
    level_kernel alone; CUDA events around 10 back-to-back launches."""
    import numpy as np
    import paper_2204_06045_b200 as q
    peak, kind = load_peaks()
    rng = np.random.default_rng(7)
    out = {"peak_GBps": peak, "peak_source": kind, "cases": []}
    for w in widths:
        a = rng.uniform(-1, 1, 1 << w) + 1j * rng.uniform(-1, 1, 1 << w)
        b = rng.uniform(-1, 1, 4) + 1j * rng.uniform(-1, 1, 4)
        sch = q.ContractionSchedule([q.Bucket([0], [q.Tensor("a", list(range(w)), a),
                                                    q.Tensor("b", [0, 1], b)])])
        plan = q.Plan.from_schedule(sch, ctx=ctx)
        plan.execute()
        _, by, ms = plan.time_level(0, 10)
        plan.close()
        gbs = by / (ms * 1e-3) / 1e9
        out["cases"].append({"bucket": f"[{w},2]->{w - 1}", "alg_bytes": by, "ms": ms,
                             "GBps": gbs, "frac": gbs / peak})
    return out


def cpu_baseline(cfg):
    """The reference's own energy_expectation on this host's cores (BASELINE.md
    section 3's "CPU best"): full C2 energies, best of 3 with the matmul backend
    and one with mixed(15), jobs = all threads, in a subprocess so that
    OPENBLAS_NUM_THREADS=1 applies.  value = the faster (~15-20 s of CPU work)."""
    code = (
        "import os,sys,json,time;sys.path.insert(0,%r);import oracle as O\n"
        "c=json.loads(%r);e=O.ref_random_regular(c['n'],c['d'],c['seed'])\n"
        "j=int(sys.argv[1]);runs=[]\n"
        "for b in ('matmul','matmul','matmul','mixed'):\n"
        "    en,w,_,_=O.ref_energy(c['n'],e,c['gammas'],c['betas'],b,threshold=15,jobs=j)\n"
        "    runs.append({'backend':b,'energy':en,'wall':w})\n"
        "print(json.dumps({'runs':runs,'m':len(e)}))\n"
    ) % (os.path.join(ROOT, "oracle"), json.dumps(cfg))
    jobs = cpu_threads()
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", code, str(jobs)], capture_output=True, text=True,
                           env=env, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        best = min(d["runs"], key=lambda x: x["wall"])
        walls = {b: [round(x["wall"], 3) for x in d["runs"] if x["backend"] == b]
                 for b in ("matmul", "mixed")}
        return {"value": d["m"] / best["wall"], "unit": "lightcones/s", "cores": jobs,
                "kind": "reference", "energy": best["energy"], "wall_s": best["wall"],
                "backend": best["backend"], "walls_s": walls,
                "sample": "full energies (all lightcones): best of 3 x matmul and 1 x mixed(15), "
                          f"jobs={jobs}, OPENBLAS_NUM_THREADS=1"}
    except Exception as ex:  # reported, not fatal
        return {"value": None, "unit": "lightcones/s", "cores": jobs, "kind": "reference",
                "sample": f"failed: {ex!r}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the single-bucket microbench")
    ap.add_argument("--no-sub", action="store_true", help="skip the C4 / c64 / multi sub-records")
    ap.add_argument("--dtype", choices=["c128", "c64"], default="c128",
                    help="c64: the optional complex64 mode (1e-5), not the headline")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = dict(CONFIGS[args.config])
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_b200(args, cfg)


if __name__ == "__main__":
    sys.exit(main())

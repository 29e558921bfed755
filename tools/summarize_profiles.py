#!/usr/bin/env python3
"""Turn a gpurun_out/<tag>/ directory (tools/gpu_check.sh output) into the
committed evidence under profiles/<tag>/:

  launches.csv            ncu launch list of one C2 step (per-launch duration,
                          DRAM read/write bytes; cold-cache, serialised)
  launch_summary.txt      per level: us, DRAM GB, GB/s; shares of the step
  ncu_widest_level.txt    key metrics + stall breakdown of the full ncu capture
                          of the widest-bucket level (level_kernel)
  bench.json / microbench.txt / pytest_gpu.txt copied verbatim
  traffic.json            DRAM bytes per step of the level kernel (read by bench.py)
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum"]


def launches(src, dst_dir):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ii, mi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "ID", "Metric Name"))
    d = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        try:
            d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
            names[int(r[ii])] = r[ki].split("(")[0].split("::")[-1]
        except ValueError:
            pass
    ids = sorted(d)
    half = ids[len(ids) // 2:]  # the profiled (second, warm) step
    tot_t = sum(d[i]["gpu__time_duration.sum"] for i in half)
    tot_b = sum(d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)
                for i in half)
    kinds = defaultdict(lambda: [0.0, 0.0])  # kernel -> [ns, DRAM bytes] per step
    for i in half:
        k = kinds[names[i].split("<")[0]]
        k[0] += d[i]["gpu__time_duration.sum"]
        k[1] += d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)
    lines = [f"launches per step: {len(half)}; step total {tot_t / 1e3:.1f} us (ncu-serialised); "
             f"DRAM {tot_b / 1e9:.3f} GB; " + "; ".join(
                 f"{k} {100 * v[0] / tot_t:.1f}% of time, {v[1] / 1e9:.3f} GB"
                 for k, v in sorted(kinds.items(), key=lambda kv: -kv[1][0])),
             "idx kernel us DRAM_MB GB/s share%"]
    for j, i in enumerate(half):
        t = d[i]["gpu__time_duration.sum"]
        b = d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)
        lines.append(f"{j} {names[i]} {t / 1e3:.1f} {b / 1e6:.1f} {b / t:.0f} {100 * t / tot_t:.2f}")
    open(os.path.join(dst_dir, "launch_summary.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"dram_bytes_per_step": {k: v[1] for k, v in kinds.items()},
               "ncu_us_per_step": {k: v[0] / 1e3 for k, v in kinds.items()},
               "source": os.path.relpath(os.path.join(dst_dir, "launches.csv"), ROOT)},
              open(os.path.join(dst_dir, "traffic.json"), "w"), indent=1)
    return lines[0]


def full_capture(rep, dst):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = [f"{h} [{units[i]}] = {vals[i]}" for i, h in enumerate(hdr) if h in KEYS]
    items = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                items.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1.0
    out.append("stall reasons (pc sampling): " + ", ".join(
        f"{h} {100 * v / tot:.1f}%" for v, h in sorted(items, reverse=True)[:8]))
    open(dst, "w").write("\n".join(out) + "\n")


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    for f in ("bench.json", "bench_reference.json", "microbench.txt", "pytest_gpu.txt", "smoke.txt",
              "launches.csv", "host.txt", "levels.txt"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    if os.path.exists(os.path.join(src, "launches.csv")):
        print(launches(os.path.join(src, "launches.csv"), dst))
    if os.path.exists(os.path.join(src, "prof_big.ncu-rep")):
        full_capture(os.path.join(src, "prof_big.ncu-rep"), os.path.join(dst, "ncu_widest_level.txt"))
    if os.path.exists(os.path.join(src, "seg.ncu-rep")):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                              os.path.join(src, "seg.ncu-rep"), "30"], capture_output=True, text=True).stdout
        open(os.path.join(dst, "ncu_seg_kernel.txt"), "w").write(out)
    if os.path.exists(os.path.join(src, "seg4.ncu-rep")):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                              os.path.join(src, "seg4.ncu-rep"), "30"], capture_output=True, text=True).stdout
        open(os.path.join(dst, "ncu_seg4_kernel.txt"), "w").write(out)
    print("wrote", dst)


if __name__ == "__main__":
    main()

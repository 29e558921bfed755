#!/usr/bin/env python3
"""Summarise one ncu report: key raw metrics, stall reasons and the hottest
source lines (stall samples / executed instructions).

  python tools/ncu_summary.py gpurun_out/<tag>/<name>.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, val = rows[0], rows[2]
    stalls = []
    for n, v in zip(hdr, val):
        if n in KEYS:
            print(f"{n} = {v}")
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                stalls.append((float(v), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in stalls) or 1.0
    print("stalls: " + ", ".join(f"{k} {100 * x / tot:.1f}%" for x, k in sorted(stalls, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    line = {}
    for r in src[3:]:
        if len(r) > 8 and r[0].isdigit():
            try:
                line[int(r[0])] = (float(r[4]), float(r[7]), r[1])
            except ValueError:
                pass
    ts = sum(v[0] for v in line.values()) or 1.0
    ti = sum(v[1] for v in line.values()) or 1.0
    for ln, v in sorted(line.items(), key=lambda kv: -kv[1][0])[:nl]:
        print(f"{ln:5d} stall {100 * v[0] / ts:5.1f}% inst {100 * v[1] / ti:5.1f}%  {v[2][:96]}")


if __name__ == "__main__":
    main()

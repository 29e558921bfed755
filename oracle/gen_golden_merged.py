#!/usr/bin/env python3
"""Golden fixtures of the MERGED path (merge_buckets, proj/src/engine.cpp:306-358)
from the UNMODIFIED reference (oracle/_ref/libqtnsim_ref.so).  TEST
INFRASTRUCTURE ONLY.  Writes tests/golden/merged.json.

Run here (where /root/reference exists):  make -C oracle ref && python oracle/gen_golden_merged.py

Per config (C1, C2, C4 of gen_golden.py):
  merged_buckets   FNV-1a 64 over every edge's merged schedule: per bucket the
                   sum vars, -2, each tensor's vars followed by -3, then -4;
                   -1 after each edge (the initial_buckets recipe of gen_golden.py)
  merged_widths    FNV-1a 64 over simulate_widths of the merged schedules, -5 per edge
  merges_applied / merges_skipped   per edge (ContractionSchedule counters)
  energy_naive / terms_naive        energy_expectation(merged=true) with the naive
                   backend (deterministic; 17 significant digits)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402
from gen_golden import CONFIGS, f17  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "merged.json")


def record(name, c, jobs):
    t0 = time.time()
    n, g, b = c["n"], c["gammas"], c["betas"]
    edges = O.ref_random_regular(n, 3, c["seed"])
    fp_b, fp_w, applied, skipped, shapes = [], [], [], [], []
    for i in range(len(edges)):
        ints, _, nb = O.ref_edge_schedule(n, edges, g, b, i, merged=True)
        sched = O.parse_schedule(ints, nb)
        for sums, ts in sched:
            fp_b += sums + [-2]
            for t in ts:
                fp_b += t + [-3]
            fp_b += [-4]
        fp_b.append(-1)
        w = [int(x) for x in O.ref_simulate_widths(n, edges, g, b, i, merged=True)]
        fp_w += w + [-5]
        ap, sk = O.ref_merge_counts(n, edges, g, b, i)
        applied.append(ap)
        skipped.append(sk)
        shapes.append(dict(n_buckets=len(sched), max_sum=max(len(s) for s, _ in sched),
                           max_width=max(w)))
    terms, wall = O.ref_edge_terms(n, edges, g, b, "naive", merged=True, jobs=jobs)
    e = 0.5 * len(edges) - 0.5 * sum(t.real for t in terms)  # engine.cpp:549-560
    e_ref, _, _, _ = O.ref_energy(n, edges, g, b, "naive", merged=True, jobs=jobs)
    assert e == e_ref, (e, e_ref)
    print(f"  {name}: merged E={e!r} applied={sum(applied)} skipped={sum(skipped)} "
          f"({time.time() - t0:.1f}s, contraction {wall:.1f}s)", flush=True)
    return dict(name=name, n=n, seed=c["seed"], gammas=g, betas=b,
                merged_buckets="%016x" % O.fnv1a_int64(fp_b),
                merged_widths="%016x" % O.fnv1a_int64(fp_w),
                merges_applied=applied, merges_skipped=skipped,
                max_sum_vars=max(s["max_sum"] for s in shapes),
                max_width=max(s["max_width"] for s in shapes),
                n_buckets=sum(s["n_buckets"] for s in shapes),
                energy_naive=f17(e),
                terms_naive=[[f17(z.real), f17(z.imag)] for z in terms])


def main():
    jobs = os.cpu_count() or 8
    out = {name: record(name, c, jobs) for name, c in CONFIGS.items()}
    with open(OUT, "w") as f:
        json.dump(out, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Per-bucket-class efficiency on the real C2 bucket shapes (tuning aid).

Takes the N largest device ops of the N=30 p=4 plan (qtng_plan_dump),
rebuilds each as a standalone bucket with the same operand bit maps and
random data, and times it alone (Plan.from_schedule + time_level) against
the HBM peak.  Classes: T1 (one operand), onebig (one operand of rank >= 12),
outer (>= 2 operands of rank >= 12).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402


def op_bytes(o):
    return 16 * (2 ** o["r"] + sum(2 ** x[0] for x in o["inputs"]))


def cls(o):
    big = [x for x in o["inputs"] if x[0] >= 12]
    if o["nt"] == 1:
        return "T1"
    return "outer" if len(big) >= 2 else ("onebig" if big else "tiny")


def bucket_of(o, rng):
    r, ns = o["r"], o["ns"]

    def vid(src):
        return 2 * (r - 1 - src) if src < 64 else 100000 + (ns - 1 - (src - 64))

    ts = []
    for rank, _init, src in o["inputs"]:
        d = rng.uniform(-1, 1, 1 << rank) + 1j * rng.uniform(-1, 1, 1 << rank)
        ts.append(q.Tensor("t", [vid(s) for s in src], d))
    return q.Bucket([100000 + k for k in range(ns)], ts)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    ctx = q.Context(0)
    peak = 6535.1
    g = q.random_regular(30, 3, 104478)
    ops = sorted(q.plan_dump(g, 4), key=op_bytes, reverse=True)[:n]
    rng = np.random.default_rng(3)
    for o in ops:
        plan = q.Plan.from_schedule(q.ContractionSchedule([bucket_of(o, rng)]), ctx=ctx)
        plan.execute()
        _, by, ms = plan.time_level(0, 10)
        plan.close()
        gbs = by / (ms * 1e-3) / 1e9
        print(json.dumps({"class": cls(o), "r": o["r"], "ns": o["ns"],
                          "ranks": [x[0] for x in o["inputs"]], "MB": round(by / 1e6, 1),
                          "us": round(ms * 1e3, 1), "GBps": round(gbs), "frac": round(gbs / peak, 3)}),
              flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Single-GPU simulation of N-GPU strong scaling: the library's LPT shards
(qtng_shard_edges, the placement of both multi-GPU drivers) for N = 1, 2, 4,
8, each planned and timed alone (graph replay) on this device; the N-GPU step
time is bounded below by the slowest shard.

  shard_sim.py [C2 | C4:<seed> ...]     (default: C2 C4:1 C4:8 C4:9)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402
from paper_2204_06045_b200 import dist  # noqa: E402

ctx = q.Context(0)
for spec in (sys.argv[1:] or ["C2", "C4:1", "C4:8", "C4:9"]):
    if spec == "C2":
        g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
    else:
        g = q.random_regular(100, 3, int(spec.split(":")[1]))
        a = q.Angles([0.30, 0.25, 0.20], [0.35, 0.30, 0.25])
    p = a.depth()
    w = q.edge_work(g, p)
    base = None
    for n in (1, 2, 4, 8):
        times = []
        for shard in dist.shards_for(q, g, p, n):
            plan = q.Plan(g, p, edges=shard, ctx=ctx)
            plan.execute(a)
            plan.run_device(3)
            times.append(plan.run_device(10) / 10)
            plan.close()
        base = base or max(times)
        print(json.dumps({"config": spec, "n": n, "max_ms": round(max(times), 4),
                          "speedup": round(base / max(times), 3),
                          "work_bound": round(float(w.sum() / max(w.max(), w.sum() / n)), 2),
                          "shard_ms": [round(t, 3) for t in times]}), flush=True)

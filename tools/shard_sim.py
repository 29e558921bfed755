#!/usr/bin/env python3
"""Single-GPU simulation of N-GPU strong scaling (tuning aid): the LPT shards
of C2 for N = 1, 2, 4, 8, each planned and timed alone on this device; the
N-GPU step time is bounded below by the slowest shard."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402
from paper_2204_06045_b200 import dist  # noqa: E402

g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
costs = q.edge_work(g, 4) if os.environ.get('SHARD_KEY', 'work') == 'work' else q.edge_costs(g, 4)
for n in (1, 2, 4, 8):
    times = []
    for shard in dist.lpt_shard(costs, n):
        plan = q.Plan(g, 4, edges=shard, ctx=ctx)
        plan.execute(a)
        plan.run_device(3)
        times.append(plan.run_device(10) / 10)
        plan.close()
    print(json.dumps({"n": n, "max_ms": max(times), "shard_ms": [round(t, 3) for t in times]}), flush=True)

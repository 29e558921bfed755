#!/usr/bin/env python3
"""C2 at N=1 and the largest 8-way shard for several QTNG_SEG_STARVED values."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys; sys.path.insert(0, %r)
import paper_2204_06045_b200 as q
from paper_2204_06045_b200 import dist
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
out = []
for edges in (None, dist.lpt_shard(q.edge_costs(g, 4), 8)[0], dist.lpt_shard(q.edge_costs(g, 4), 8)[2]):
    plan = q.Plan(g, 4, edges=edges, ctx=ctx)
    t = plan.execute(a); plan.run_device(3)
    out.append(round(plan.run_device(10) / 10, 4)); plan.close()
print(out)
''' % ROOT
for v in ("0", "256", "1024", "4096", "16384"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, QTNG_SEG_STARVED=v),
                       capture_output=True, text=True, timeout=300)
    print("starved", v, r.stdout.strip(), r.stderr[-200:], flush=True)

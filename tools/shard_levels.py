#!/usr/bin/env python3
"""Per-level device time of the slowest 8-way LPT shard of C2 (eager
profile; where the multi-GPU latency floor goes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q
from paper_2204_06045_b200 import dist

g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
shards = dist.shards_for(q, g, 4, 8)
best = None
for s in shards:
    p = q.Plan(g, 4, edges=s, ctx=ctx)
    p.execute(a); p.run_device(3)
    t = p.run_device(20) / 20
    if best is None or t > best[0]:
        best = (t, s)
    p.close()
t, s = best
plan = q.Plan(g, 4, edges=s, ctx=ctx)
for _ in range(3):
    plan.profile(a)
lv, kms = plan.level_ms(), plan.level_kernel_ms()
info = plan.info()
print(f"slowest shard: {len(s)} lightcones, graph replay {t:.3f} ms, eager levels sum {1e3 * lv.sum():.1f} us, "
      f"{info.n_levels} levels, {info.kernels_per_run} kernels")
print("level  us  level_k  seg_k  seg4_k")
for L in range(len(lv)):
    print(f"{L:4d} {1e3 * lv[L]:7.1f} {1e3 * kms[L, 0]:7.1f} {1e3 * kms[L, 2]:7.1f} {1e3 * kms[L, 3]:7.1f}")

#!/usr/bin/env python3
"""Per-level device times of one N-GPU LPT shard of C2 (tuning aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402
from paper_2204_06045_b200 import dist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
shard = dist.lpt_shard(q.edge_costs(g, 4), n)[0]
plan = q.Plan(g, 4, edges=shard)
for _ in range(3):
    plan.profile(a)
lv, k = plan.level_ms(), plan.level_kernel_ms()
print("edges", len(shard), "levels", len(lv), "graph ms", plan.run_device(10) / 10)
for L in range(len(lv)):
    print(f"{L:3d} {1e3 * lv[L]:7.1f} level_k {1e3 * k[L, 0]:6.1f} seg_k {1e3 * k[L, 2]:6.1f}")

#!/usr/bin/env python3
"""Per-level device time of the C2 plan (tuning aid, not a bench number):
level events, per-kernel-kind events, and the segment work of each level."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402

g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
plan = q.Plan(g, 4)
for _ in range(3):
    plan.profile(a)
lv, kms = plan.level_ms(), plan.level_kernel_ms()
segs = q.plan_segments(g, 4)
by = collections.defaultdict(list)
for s in segs:
    by[s["level"]].append(s)
print("level  ms   level_k  seg_k  | segs  x1_elems  tiles")
for L in range(len(lv)):
    ss = by.get(L, [])
    x1 = sum(2 ** (s["ry"] + s["L"] - 1) for s in ss)
    tiles = sum(2 ** (s["ry"] - s["cy"]) for s in ss)
    print(f"{L:4d} {1e3 * lv[L]:7.1f} {1e3 * kms[L, 0]:7.1f} {1e3 * (kms[L, 2] + kms[L, 3]):7.1f} | {len(ss):4d} {x1:9.3g} {tiles:6d}")
print("total", 1e3 * lv.sum(), plan.kernel_ms())

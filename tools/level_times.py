#!/usr/bin/env python3
"""Per-level device time of the C2 plan for every libqtng variant in
build/variants (tuning aid): level ms and its level/seg kernel split."""
import glob, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r)
import paper_2204_06045_b200 as q
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
plan = q.Plan(g, 4)
for _ in range(5): plan.profile(a)
lv, k = plan.level_ms(), plan.level_kernel_ms()
print("step", round(plan.run_device(20) / 20, 4))
print("level_ms ", " ".join("%%.1f" %% (1e3 * x) for x in lv))
print("level_k  ", " ".join("%%.1f" %% (1e3 * x) for x in k[:, 0]))
print("seg_k    ", " ".join("%%.1f" %% (1e3 * x) for x in k[:, 2]))
''' % ROOT
for so in sorted(glob.glob(os.path.join(ROOT, "build/variants/*.so"))):
    r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, QTNG_LIB_PATH=so),
                       capture_output=True, text=True, timeout=300)
    print(os.path.basename(so), flush=True)
    print(r.stdout.strip() or r.stderr[-500:], flush=True)

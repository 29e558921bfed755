#!/usr/bin/env python3
"""Kernel variant sweep on the GPU (tuning only, not a bench number):
for each libqtng variant x planner switch, C2 device ms/step and the widest level."""
import glob, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_2204_06045_b200 as q
g = q.random_regular(30, 3, 104478); a = q.Angles([0.30,0.25,0.20,0.15],[0.35,0.30,0.25,0.20])
ctx = q.Context(0); plan = q.Plan(g, 4, ctx=ctx)
try:
    t = plan.profile(a); e = 0.5*g.m - 0.5*float(np.sum(t.real))
except Exception as ex:  # timing experiments may compute garbage
    e = repr(ex)[:60]
for _ in range(3): plan.run_device(1)
ms = plan.run_device(20) / 20
try:
    plan.profile(a)
except Exception:
    pass
lv = plan.level_ms()
L, by, lms = plan.time_level(-1, 20)
print(json.dumps(dict(ms_step=ms, level_sum=float(lv.sum()), big_level=L, big_gbs=by/lms/1e6, energy=e,
                      top=[round(float(x),1) for x in sorted(lv*1e3)[-6:]])))
''' % ROOT
# env sweeps: "NAME=v1,v2;NAME2=..." (default: one run per variant)
sweep = [[]]
for part in (sys.argv[1] if len(sys.argv) > 1 else "").split(";"):
    if "=" in part:
        k, vs = part.split("=", 1)
        sweep = [s + [(k, v)] for s in sweep for v in vs.split(",")]
for so in sorted(glob.glob(os.path.join(ROOT, "build/variants/*.so"))):
    for combo in sweep:
        env = dict(os.environ, QTNG_LIB_PATH=so, **dict(combo))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        line = (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1]
        print(os.path.basename(so), " ".join(f"{k}={v}" for k, v in combo), line, flush=True)

#!/usr/bin/env python3
"""e2e wall time of energy_expectation for several pipelining lane counts
(QTNG_PIPELINE, read once per process -> one subprocess each)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, time; sys.path.insert(0, %r)
import paper_2204_06045_b200 as q
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
for _ in range(5): r = q.energy_expectation(g, a, q.GpuBackend(ctx))
ts = []
for _ in range(20):
    t0 = time.perf_counter(); r = q.energy_expectation(g, a, q.GpuBackend(ctx)); ts.append(time.perf_counter() - t0)
ts.sort(); print("median ms %%.3f min %%.3f energy %%r" %% (1e3 * ts[10], 1e3 * ts[0], r.energy))
''' % ROOT
sweep = [dict(QTNG_PIPELINE=k, QTNG_PIPELINE_ORDER=o) for o in ("0", "1") for k in ("1", "2", "3", "4")]
if len(sys.argv) > 1 and sys.argv[1] == "split":  # chunk fractions, two passes
    splits = [("3", "1,1,1"), ("3", "0.45,0.35,0.2"), ("3", "0.4,0.35,0.25"), ("3", "0.5,0.3,0.2"),
              ("2", "0.6,0.4"), ("2", "0.7,0.3"), ("4", "0.35,0.3,0.2,0.15"), ("3", "0.3,0.35,0.35")]
    sweep = [dict(QTNG_PIPELINE=k, QTNG_PIPELINE_SPLIT=f) for _ in range(2) for k, f in splits]
if len(sys.argv) > 1 and sys.argv[1] == "pool":  # host pool sizes, 3 repetitions each
    sweep = [dict(QTNG_POOL_THREADS=t) for t in ("16", "14", "12", "8") for _ in range(3)]
for env in sweep:
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=300)
    print(env, out.stdout.strip(), out.stderr[-200:], flush=True)

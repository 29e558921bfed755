#!/usr/bin/env python3
"""Short, deterministic launch sequence for ncu (never a bench number).

  profile_step.py levels        print the number of level_kernel launches per step
  profile_step.py step          warm-up step + 1 profiled step (launch list)
  profile_step.py big           warm-up step + the widest-bucket level once more
                                (ncu -k regex:level_kernel -s <levels+1> -c 1)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402

cfg = os.environ.get("QTNG_CFG", "C2")
if cfg == "C2":
    g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
else:
    g, a = q.random_regular(100, 3, 1), q.Angles([0.30, 0.25, 0.20], [0.35, 0.30, 0.25])
ctx = q.Context(0)
plan = q.Plan(g, a.depth(), ctx=ctx)
mode = sys.argv[1] if len(sys.argv) > 1 else "step"
if mode == "levels":
    print(plan.info().n_levels)
    sys.exit(0)
plan.execute(a)
if mode == "step":
    plan.execute(a)
else:
    plan.time_level(-1, 1)

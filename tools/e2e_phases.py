#!/usr/bin/env python3
"""Host/device phase times of energy_expectation (QTNG_TIMING=1, tuning aid)."""
import os
import sys
os.environ.setdefault("QTNG_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402

g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
for _ in range(8):
    q.energy_expectation(g, a, q.GpuBackend(ctx))
print("threads", os.cpu_count())

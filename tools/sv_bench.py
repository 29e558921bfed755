#!/usr/bin/env python3
"""Device state-vector oracle timing (tuning aid): C2 (30 qubits, p=4) energy
by brute force, wall time around the synchronous call, and the HBM traffic the
passes imply (3 tile passes per layer, read+write; 3 expectation reads)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
g = q.random_regular(n, 3, 104478 if n == 30 else 7)
a = q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
ctx = q.Context(0)
q.statevector_energy(g, a, cap=n, ctx=ctx)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    e, _ = q.statevector_energy(g, a, cap=n, ctx=ctx)
    ts.append(time.perf_counter() - t0)
groups = len(range(n, 0, -9)) if n > 12 else 1
passes = 4 * (3 if n >= 22 else (2 if n > 12 else 1))
bytes_ = (passes * 2 + 3 + 1) * 16 * 2 ** n
t = min(ts)
print(json.dumps({"n": n, "energy": e, "s": t, "GBps": bytes_ / t / 1e9, "bytes": bytes_}))

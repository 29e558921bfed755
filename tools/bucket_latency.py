#!/usr/bin/env python3
"""Per-call latency of the single-bucket drop-in (qtng_contract_bucket, what
qtng::GpuBackend::contract calls for every bucket) for C2-like small buckets,
with QTNG_TIMING-style host phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2204_06045_b200 as q

ctx = q.Context(0)
rng = np.random.default_rng(1)
for nvars, nt in ((4, 3), (8, 3), (12, 3), (16, 3), (20, 2)):
    vs = list(range(nvars))
    ts = []
    for t in range(nt):
        v = vs if t == 0 else sorted(rng.choice(vs, size=min(2, nvars), replace=False).tolist())
        d = rng.uniform(-1, 1, 1 << len(v)) + 1j * rng.uniform(-1, 1, 1 << len(v))
        ts.append(q.Tensor("t", v, d))
    b = q.Bucket([0], ts)
    for _ in range(20):
        q.contract_bucket(b, ctx)
    n = 200 if nvars < 16 else 50
    t0 = time.perf_counter()
    for _ in range(n):
        q.contract_bucket(b, ctx)
    print(f"bucket vars={nvars} members={nt}: {1e6 * (time.perf_counter() - t0) / n:.1f} us/call", flush=True)

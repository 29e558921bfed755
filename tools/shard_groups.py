#!/usr/bin/env python3
"""Experiment: the 8-way shard floor is the per-level tail (a level waits for
its slowest tile, and a small shard cannot fill the device).  Split the
slowest shard's lightcones into k independent level-synchronous programs
(one context each, run concurrently) so one group's tail overlaps another
group's work.  Prints the slowest shard alone vs its k-group concurrent wall.

  shard_groups.py [C2 | C4:<seed> ...] [--n 8]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2204_06045_b200 as q  # noqa: E402
from paper_2204_06045_b200 import dist  # noqa: E402

args = [x for x in sys.argv[1:] if not x.startswith("--")]
n_gpu = 8
if "--n" in sys.argv:
    n_gpu = int(sys.argv[sys.argv.index("--n") + 1])
    args = [x for x in args if x != str(n_gpu)]
N = 50
for spec in (args or ["C2", "C4:9"]):
    if spec == "C2":
        g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
    else:
        g = q.random_regular(100, 3, int(spec.split(":")[1]))
        a = q.Angles([0.30, 0.25, 0.20], [0.35, 0.30, 0.25])
    p = a.depth()
    w = q.edge_work(g, p)
    ctx = q.Context(0)
    worst = None
    for shard in dist.shards_for(q, g, p, n_gpu):
        plan = q.Plan(g, p, edges=shard, ctx=ctx)
        plan.execute(a)
        plan.run_device(3)
        t = plan.run_device(N) / N
        plan.close()
        if worst is None or t > worst[0]:
            worst = (t, list(shard))
    t1, shard = worst
    print(f"{spec} n={n_gpu}: slowest shard {len(shard)} lightcones, alone {t1:.3f} ms", flush=True)
    for k in sorted({2, 3, 4, len(shard)}):
        if k > len(shard):
            continue
        # LPT of the shard's lightcones over k groups
        order = sorted(shard, key=lambda e: -w[e])
        groups, load = [[] for _ in range(k)], [0.0] * k
        for e in order:
            i = int(np.argmin(load))
            groups[i].append(e)
            load[i] += w[e]
        ctxs = [q.Context(0) for _ in range(k)]
        plans = [q.Plan(g, p, edges=sorted(gr), ctx=c) for gr, c in zip(groups, ctxs)]
        for pl in plans:
            pl.execute(a)
            pl.run_device(3)
        alone = [pl.run_device(N) / N for pl in plans]

        def run(pl):
            pl.run_device(N)
        best = None
        for _ in range(3):
            th = [threading.Thread(target=run, args=(pl,)) for pl in plans]
            t0 = time.perf_counter()
            for t in th:
                t.start()
            for t in th:
                t.join()
            wall = (time.perf_counter() - t0) * 1e3 / N
            best = wall if best is None else min(best, wall)
        print(f"  k={k}: groups alone {['%.3f' % x for x in alone]} ms; concurrent wall {best:.3f} ms "
              f"({t1 / best:.2f}x vs one program)", flush=True)
        for pl in plans:
            pl.close()

#!/usr/bin/env python3
"""Experiment: do independent lightcone groups, each its own level-synchronous
program on its own context (streams), overlap on the device better than one
program over all lightcones?  (The level barrier couples every lightcone.)"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2204_06045_b200 as q

g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
N = 20
base = q.Context(0)
plan = q.Plan(g, 4, ctx=base)
plan.execute(a)
plan.run_device(5)
print("one program: %.3f ms" % (plan.run_device(N) / N))
w = q.edge_work(g, 4)
for k in (2, 3, 4):
    own = q.shard_edges(g, 4, k)
    ctxs = [q.Context(0) for _ in range(k)]
    plans = [q.Plan(g, 4, edges=[int(i) for i in np.nonzero(own == r)[0]], ctx=ctxs[r]) for r in range(k)]
    for p in plans:
        p.execute(a)
        p.run_device(3)
    alone = [p.run_device(N) / N for p in plans]
    ts = []
    def run(p):
        p.run_device(N)
    th = [threading.Thread(target=run, args=(p,)) for p in plans]
    t0 = time.perf_counter()
    for t in th: t.start()
    for t in th: t.join()
    wall = (time.perf_counter() - t0) * 1e3 / N
    print("k=%d groups: alone %s ms; concurrent wall %.3f ms/step" % (k, ["%.3f" % x for x in alone], wall))

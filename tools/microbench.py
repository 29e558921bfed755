#!/usr/bin/env python3
"""C3 microbenchmark (BASELINE.json configs[2]): single wide buckets vs the HBM roofline.

(i)  calibrate()'s synthetic bucket (proj/src/engine.cpp:371-390): a rank-w
     tensor on vars 0..w-1 times a rank-2 tensor on {0,1}, summing var 0 (the
     MSB): [w, 2] -> w-1, algorithmic bytes 16*(2^w + 4 + 2^(w-1)).
(ii) the widest real buckets of the N=30 p=4 energy: the level holding each
     of the two widest lightcones' widest bucket, timed in isolation.
Device time = CUDA events around back-to-back launches of the level kernel
on the library stream (warm).  Prints one JSON line per case.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def synthetic(w, ctx, rng):
    a = rng.uniform(-1, 1, 1 << w) + 1j * rng.uniform(-1, 1, 1 << w)
    b = rng.uniform(-1, 1, 4) + 1j * rng.uniform(-1, 1, 4)
    sch = q.ContractionSchedule([q.Bucket([0], [q.Tensor("a", list(range(w)), a),
                                                q.Tensor("b", [0, 1], b)])])
    plan = q.Plan.from_schedule(sch, ctx=ctx)
    plan.execute()
    lv, by, ms = plan.time_level(0, 10)
    plan.close()
    return by, ms


def main():
    ctx = q.Context(0)
    pk = peak()
    rng = np.random.default_rng(7)
    widths = [int(x) for x in sys.argv[1:]] or list(range(20, 29))
    for w in widths:
        by, ms = synthetic(w, ctx, rng)
        gbs = by / (ms * 1e-3) / 1e9
        print(json.dumps({"case": f"synthetic [{w},2]->{w - 1}", "alg_bytes": by, "ms": ms,
                          "GBps": gbs, "frac": gbs / pk}), flush=True)
    g = q.random_regular(30, 3, 104478)
    a = q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
    costs = q.edge_costs(g, 4)
    for e in np.argsort(-costs)[:2]:
        plan = q.Plan(g, 4, edges=[int(e)], ctx=ctx)
        plan.execute(a)
        lv, by, ms = plan.time_level(-1, 10)
        gbs = by / (ms * 1e-3) / 1e9
        print(json.dumps({"case": f"C2 edge {g.edges[e].tolist()} widest-bucket level {lv}",
                          "alg_bytes": by, "ms": ms, "GBps": gbs, "frac": gbs / pk}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()

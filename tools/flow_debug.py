import os, sys
os.environ["QTNG_FLOW"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06045_b200 as q
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
plan = q.Plan(g, 4)
plan.execute(a)
print("units", plan.info().n_device_ops + plan.info().n_segments, "ms", plan.run_device(1), flush=True)

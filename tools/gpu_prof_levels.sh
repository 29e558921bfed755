cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/p1; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py step > $O/ncu.txt 2>&1
python - > $O/levels.txt 2>&1 <<'PY'
import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2204_06045_b200 as q
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
plan = q.Plan(g, 4)
for _ in range(3): plan.profile(a)
print('device ms', plan.last_device_ms)
print(' '.join('%.1f' % (1000 * x) for x in plan.level_ms()))
PY

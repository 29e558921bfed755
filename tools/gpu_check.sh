#!/bin/bash
# One gpurun call = the round's evidence: smoke, GPU parity tests, bench (both
# arms), microbench, ncu launch list of one step, full ncu capture of the
# biggest seg_kernel launch.   usage: tools/gpu_check.sh <tag> [skip-tests]
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-run}
O=gpurun_out/$T
mkdir -p $O
{ nvidia-smi -L; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; } > $O/host.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
fi
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err
timeout 300 python tools/microbench.py > $O/microbench.txt 2>&1
timeout 120 python - > $O/levels.txt 2>&1 <<'PY'
import sys
sys.path.insert(0, '.')
import paper_2204_06045_b200 as q
g, a = q.random_regular(30, 3, 104478), q.Angles([0.30, 0.25, 0.20, 0.15], [0.35, 0.30, 0.25, 0.20])
plan = q.Plan(g, 4)
for _ in range(3): plan.profile(a)
print('levels', plan.info().n_levels, 'kernel_ms', plan.kernel_ms())
print(' '.join('%.1f' % (1000 * x) for x in plan.level_ms()))
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py step > $O/ncu.txt 2>&1
# skip count of the longest seg_kernel launch of the profiled (second) step
SEGSKIP=$(python - "$O/launches.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ii, ki, mi, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
t = {}
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum" and "seg_kernel" in r[ki]:
        t[int(r[ii])] = float(r[vi].replace(",", ""))
ids = sorted(t); half = len(ids) // 2
best = max(range(half, len(ids)), key=lambda k: t[ids[k]])
print(best)
PY
)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s ${SEGSKIP:-27} -c 1 -o $O/seg python tools/profile_step.py step >> $O/ncu.txt 2>&1
echo "ncu rc=$?" >> $O/ncu.txt
# the longest seg4_kernel (quad tiles) launch of the profiled step
SEG4SKIP=$(python - "$O/launches.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ii, ki, mi, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
t = {}
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum" and "seg4_kernel" in r[ki]:
        t[int(r[ii])] = float(r[vi].replace(",", ""))
ids = sorted(t); half = len(ids) // 2
print(max(range(half, len(ids)), key=lambda k: t[ids[k]]) if ids else -1)
PY
)
if [ "${SEG4SKIP:--1}" -ge 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg4_kernel -s $SEG4SKIP -c 1 -o $O/seg4 python tools/profile_step.py step >> $O/ncu.txt 2>&1
  echo "ncu seg4 rc=$?" >> $O/ncu.txt
fi

#!/bin/bash
# Full ncu capture of the N-th launch (0-based, second step) of kernel KRE.
#   usage: KRE=seg_kernel tools/gpu_ncu_nth.sh <tag> <n>
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-ncu}; N=${2:-4}; O=gpurun_out/$T; mkdir -p $O
K=${KRE:-seg_kernel}
PER=$(python - <<PY
import subprocess, sys
PY
)
# launches of K per step: count from a launch list
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:$K --log-file $O/list.csv python tools/profile_step.py step > /dev/null 2>&1
SKIP=$(python - "$O/list.csv" $N <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
n = len(rows) - 1
print(n // 2 + int(sys.argv[2]))
PY
)
echo "skip=$SKIP" > $O/ncu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o $O/k python tools/profile_step.py step >> $O/ncu.txt 2>&1
echo "ncu rc=$?" >> $O/ncu.txt

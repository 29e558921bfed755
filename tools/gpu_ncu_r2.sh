#!/bin/bash
# ncu evidence: launch list of one C2 step, then a --set full capture of the
# longest seg_kernel launch of the second step.   usage: tools/gpu_ncu_r2.sh <tag>
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-ncu}; O=gpurun_out/$T; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py step > $O/ncu.txt 2>&1
SEGSKIP=$(python - "$O/launches.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ii, ki, mi, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
t = {}
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum" and (__import__("os").environ.get("KRE","seg_kernel")) in r[ki]:
        t[int(r[ii])] = float(r[vi].replace(",", ""))
ids = sorted(t); half = len(ids) // 2
print(max(range(half, len(ids)), key=lambda k: t[ids[k]]))
PY
)
echo "segskip=$SEGSKIP" >> $O/ncu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-seg_kernel} -s ${SEGSKIP:-30} -c 1 -o $O/seg python tools/profile_step.py step >> $O/ncu.txt 2>&1
echo "ncu rc=$?" >> $O/ncu.txt

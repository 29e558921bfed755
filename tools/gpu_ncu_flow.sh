#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-pf}; O=gpurun_out/$T; mkdir -p $O
QTNG_FLOW=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -s 1 -c 1 -o $O/flow python tools/profile_step.py step > $O/ncu.txt 2>&1
echo "rc=$?" >> $O/ncu.txt

#!/bin/bash
# Full ncu capture of one level_kernel launch (skip S matching launches).
cd "${GRAFT_REPO_ROOT:-.}"
S=${1:-0}; T=${2:-pl}; O=gpurun_out/$T; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_kernel -s $S -c 1 -o $O/lvl python tools/profile_step.py step > $O/ncu.txt 2>&1
echo "rc=$?" >> $O/ncu.txt

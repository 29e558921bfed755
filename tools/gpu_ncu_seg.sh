#!/bin/bash
# Full ncu capture of one seg_kernel launch (skip S launches; default: the 10th of the 2nd step).
cd "${GRAFT_REPO_ROOT:-.}"
S=${1:-27}; T=${2:-p2}; O=gpurun_out/$T; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s $S -c 1 -o $O/seg python tools/profile_step.py step > $O/ncu.txt 2>&1
echo "rc=$?" >> $O/ncu.txt

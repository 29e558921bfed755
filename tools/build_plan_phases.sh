#!/bin/bash
# build_plan pass times (QTNG_TIMING=2) of the one-shot energy's chunks for
# several pool sizes (host tuning aid).   usage: tools/build_plan_phases.sh <tag>
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-bp}; mkdir -p $O
for t in 14 8 4 1; do
  QTNG_POOL_THREADS=$t QTNG_TIMING=2 timeout 120 python tools/e2e_phases.py > $O/phases_$t.txt 2>&1
  echo "threads $t" >> $O/summary.txt
  tail -150 $O/phases_$t.txt | awk '{k=$1" "$2; v[k]+=$3; n[k]++} END {for (k in v) printf "  %-34s %.3f\n", k, v[k]/n[k]}' | sort >> $O/summary.txt
done

#!/bin/bash
# Bench-only A/B of environment settings, two interleaved passes (noise check).
#   usage: tools/gpu_sweep.sh <tag> "ENV1=.. ENV2=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-.}"
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for pass in 1 2; do
  for E in "$@"; do
    env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c3 --no-sub > $O/b.json 2>> $O/err.txt
    python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('BENCH', '$E', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],3))" >> $O/sweep.txt
  done
done

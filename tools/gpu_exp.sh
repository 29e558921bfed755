#!/bin/bash
# A/B experiment: per-level kernel times under several env settings + bench value.
#   usage: tools/gpu_exp.sh <tag> "ENV1=.. ENV2=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-.}"
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
i=0
for E in "$@"; do
  echo "== $E" >> $O/exp.txt
  env $E timeout 300 python tools/level_report.py >> $O/exp.txt 2>&1
  env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c3 --no-sub > $O/bench_$i.json 2>> $O/exp.txt
  python -c "import json,sys; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); print('BENCH', '$E', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'])" >> $O/exp.txt
  i=$((i+1))
done

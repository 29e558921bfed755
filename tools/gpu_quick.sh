#!/bin/bash
# Quick GPU iteration: parity tests, bench (no CPU baseline), class bench A/B.
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-quick}; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
QTNG_OUTER=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_noouter.json 2>> $O/bench.err
timeout 600 python tools/classbench.py 24 > $O/classbench.txt 2>&1

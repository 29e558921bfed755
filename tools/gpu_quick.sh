#!/bin/bash
# Quick GPU iteration: parity tests, bench with and without chain fusion.
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-quick}; O=gpurun_out/$T; mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
QTNG_FUSE=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_nofuse.json 2>> $O/bench.err

#!/bin/bash
# Round-2 GPU iteration: smoke, full -m gpu suite (or a -k filter), one bench line.
#   usage: tools/gpu_r2.sh <tag> [pytest -k expr]
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-r2}; O=gpurun_out/$T; mkdir -p $O
nvidia-smi -L > $O/host.txt 2>&1; nproc >> $O/host.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 900 python -m pytest tests -m gpu -q $K > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err

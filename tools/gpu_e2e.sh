#!/bin/bash
# e2e phases of the one-shot energy on the GPU box (host timings + lane sweep).
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-e2e}; O=gpurun_out/$T; mkdir -p $O
nproc > $O/host.txt
QTNG_TIMING=1 timeout 120 python tools/e2e_phases.py > $O/phases.txt 2>&1
QTNG_TIMING=2 timeout 120 python tools/e2e_phases.py > $O/phases2.txt 2>&1
timeout 300 python tools/e2e_sweep.py > $O/sweep.txt 2>&1

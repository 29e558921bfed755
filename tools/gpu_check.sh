#!/bin/bash
# One gpurun call: smoke, GPU parity tests, bench, ncu launch list + full capture
# of the widest-bucket level.   usage: tools/gpu_check.sh <tag> [skip-tests]
cd "${GRAFT_REPO_ROOT:-.}"
T=${1:-run}
O=gpurun_out/$T
mkdir -p $O
{ nvidia-smi -L; nproc; } > $O/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
fi
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python tools/microbench.py > $O/microbench.txt 2>&1
L=$(timeout 120 python tools/profile_step.py levels 2>/dev/null | tail -1)
echo "levels=$L" > $O/ncu.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py step >> $O/ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_kernel -s $((L+1)) -c 1 -o $O/prof_big python tools/profile_step.py big >> $O/ncu.txt 2>&1
echo "ncu rc=$?" >> $O/ncu.txt

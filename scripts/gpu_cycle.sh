#!/bin/bash
# One GPU round trip: parity tests, bench, ncu launch list, ncu full capture of a kernel.
# usage: scripts/gpu_cycle.sh TAG [kernel-regex] [bench args...]
TAG=${1:-dev}; KREGEX=${2:-mas_climb}; shift 2 2>/dev/null
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv,noheader > gpurun_out/gpu_$TAG.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
if [ -n "$KREGEX" ] && [ "$KREGEX" != "none" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 -o gpurun_out/prof_$TAG python bench.py --profile --ciphers 2000 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi

#!/bin/bash
# Quick GPU iteration: parity tests, a short bench (no CPU leg), optional ncu full capture.
# usage: scripts/gpu_quick.sh TAG [kernel-regex|none] [bench args...]
TAG=${1:-dev}; KREGEX=${2:-none}; shift 2 2>/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('value %.4g e2e %.4g frac %.3f clk %s'%(d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks']))"
if [ "$KREGEX" != "none" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 -o gpurun_out/prof_$TAG python bench.py --profile --ciphers 2000 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi

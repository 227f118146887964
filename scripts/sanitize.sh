#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tests/tools/sanitize_smoke.py
# usage: scripts/sanitize.sh OUT
OUT=${1:-gpurun_out/sanitizer.txt}; mkdir -p $(dirname $OUT)
echo "compute-sanitizer on tests/tools/sanitize_smoke.py (every climb kernel incl. the per-lane SCT parity/fast kernels and the SCT latency kernels: two-SM pair, one-CTA chain, replay), one B200" > $OUT
for tool in memcheck racecheck synccheck; do
  echo "" >> $OUT; echo "== $tool" >> $OUT
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tests/tools/sanitize_smoke.py 2>&1 | grep -v "^=========$" | tail -8 >> $OUT
done
cat $OUT

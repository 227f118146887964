#!/bin/bash
# Round-end measurement on one B200: GPU tests, smoke, the default bench line (CPU port over
# all 10k ciphertexts + configs block), the reference arm, the ncu launch list and a full
# ncu capture of the headline kernel.  usage: scripts/final_measure.sh TAG
TAG=${1:-final}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
# the reference's own test-suite against the aliased engine (staged by run_reference_suite.py --stage)
if [ -d oracle/_ref/pkg/tests ]; then timeout 600 python tests/tools/run_reference_suite.py --run > /dev/null 2>&1; echo "refsuite rc=$?"; cp gpurun_out/reference_suite.txt gpurun_out/reference_suite_$TAG.txt; tail -1 gpurun_out/reference_suite_$TAG.txt; fi
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile > /dev/null 2>&1
bash scripts/ncu_capture.sh ${TAG}_dform mas_climb_dform 1280000000 -- python bench.py --profile --ciphers 2000
python scripts/ncu_summary.py $TAG 1280000000 $TAG > /dev/null; cp profiles/${TAG}_launches.txt profiles/${TAG}_bench.json gpurun_out/ 2>/dev/null
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json")); r = json.load(open("gpurun_out/ref_$TAG.json"))
print("value %.4g e2e %.4g ref %.4g e2e-ratio %.1f clocks %s" % (d["value"], d["e2e"]["value"], r["value"], d["e2e"]["value"] / r["value"], d["clocks"]))
print("agreement", d["cpu_baseline"]["agreement"], "curves equal:", d["success_by_len"] == r["success_by_len"] == d["cpu_baseline"]["success_by_len"])
print("configs wall", d["configs"]["wall_s"], {k: (v["evals_per_s"] if isinstance(v, dict) and "evals_per_s" in v else None) for k, v in d["configs"].items() if k != "wall_s"})
PY

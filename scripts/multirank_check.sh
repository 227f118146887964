#!/bin/bash
# Exercise bench.py's multi-rank paths on a 1-GPU box:
#  (a) a plain `--gpus 2` launch must refuse to run on one GPU;
#  (b) the plain launcher and (c) torchrun, both with the ranks sharing the GPU over gloo
#      (CCG_BENCH_SHARE_GPU=1 CCG_BENCH_BACKEND=gloo), must print one line with n_gpus: 2.
# usage: scripts/multirank_check.sh TAG
TAG=${1:-dev}; mkdir -p gpurun_out; OUT=gpurun_out/multirank_$TAG.log
ARGS="--ciphers 2000 --steps 3 --warmup 3 --no-cpu --no-configs"
{
echo "== (a) python bench.py --gpus 2 (one visible GPU)"
timeout 300 python bench.py --gpus 2 $ARGS; echo "rc=$?"
echo "== (b) CCG_BENCH_SHARE_GPU=1 CCG_BENCH_BACKEND=gloo python bench.py --gpus 2"
CCG_BENCH_SHARE_GPU=1 CCG_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 $ARGS; echo "rc=$?"
echo "== (c) same, under python -m torch.distributed.run --nproc-per-node 2"
CCG_BENCH_SHARE_GPU=1 CCG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 $ARGS; echo "rc=$?"
echo "== (d) reference arm, plain --gpus 2"
timeout 300 python bench.py --impl reference --gpus 2 --ciphers 200 --steps 2 --warmup 1; echo "rc=$?"
} > $OUT 2>&1
grep -E "^==|^rc=|n_gpus|refusing" $OUT | cut -c1-200

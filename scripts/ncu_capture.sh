#!/bin/bash
# ncu --set full capture of one kernel launch, summarised ON the GPU box (the raw report can
# exceed gpurun's 64 MiB copy-back limit): writes gpurun_out/NAME_ncu.txt and removes the report.
# usage: [SKIP=n] scripts/ncu_capture.sh NAME KERNEL_REGEX TRIES_IN_CAPTURE -- command...
# (SKIP: matching launches to skip first, e.g. a warm-up launch of another size)
NAME=$1; KRE=$2; TRIES=$3; shift 4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s ${SKIP:-0} -c 1 \
  -o gpurun_out/prof_$NAME "$@" > gpurun_out/ncu_$NAME.log 2>&1
tail -1 gpurun_out/ncu_$NAME.log
python scripts/ncu_summary.py $NAME $TRIES $NAME > /dev/null && cp profiles/${NAME}_ncu.txt gpurun_out/
ncu -i gpurun_out/prof_$NAME.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/src_$NAME.csv.gz
rm -f gpurun_out/prof_$NAME.ncu-rep

#!/bin/bash
# ncu --set full (warm L2: --cache-control none) of kernels matching KREGEX in the bench step.
# Usage: profiles/run_ncu_warm.sh TAG KREGEX COUNT "<bench args>"
set -e
TAG=$1; KRE=$2; CNT=${3:-4}; ARGS=$4
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline $ARGS"
$CMD > gpurun_out/wplain_$TAG.json 2> gpurun_out/wplain_$TAG.err
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"$KRE" \
    -s 60 -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/wncu_$TAG.log 2>&1

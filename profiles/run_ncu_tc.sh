#!/bin/bash
# ncu --set full of selected kernels in the precision=1 (tcgen05) bench step. Usage: TAG KREGEX [COUNT]
set -e
TAG=${1:-tc}; KRE=${2:-k_tc_fwd}; CNT=${3:-4}
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline --precision 1"
$CMD > gpurun_out/ncu_plain_$TAG.json 2> gpurun_out/ncu_plain_$TAG.err
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 20 -c $CNT \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1

#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU). Usage: profiles/run_ncu.sh TAG KREGEX
# 1) plain run of the exact command, 2) per-launch device times (cold-cache, serialised),
# 3) one --set full capture of the kernels matching KREGEX.
set -e
TAG=${1:-r01}; KRE=${2:-k_gconv_fwd}
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$TAG.json 2> gpurun_out/ncu_plain_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 40 -c 3 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1

#!/bin/bash
# Per-launch device times of one bench step (warm L2: --cache-control none), plain run first.
# Usage: profiles/run_launches.sh TAG "<bench args>"
set -e
TAG=$1; ARGS=$2
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline $ARGS"
$CMD > gpurun_out/lplain_$TAG.json 2> gpurun_out/lplain_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 4000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/lncu_$TAG.log 2>&1

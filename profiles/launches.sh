#!/bin/bash
# Serialized per-launch device times (ncu, cold cache) of two eager steps at a workload's shapes,
# after the plain command exits 0.  Usage: profiles/launches.sh CONFIG TAG
set -e
CMD="python profiles/prof_step.py --config ${1:-pems} --steps 2"
$CMD > gpurun_out/${2}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${2}_launches.csv $CMD > gpurun_out/${2}_ncu_launch.log 2>&1

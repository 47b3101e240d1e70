#!/bin/bash
# ncu --set full of one staged-SpMM launch (both variants) at a workload's shapes (one GPU).
set -e
CFG=${1:-pems}; T=${2:-spmm}
CMD="python profiles/prof_step.py --config $CFG --steps 1"
$CMD > gpurun_out/${T}_plain.log 2>&1
PGTI_SPMM_NOPIPE=1 $CMD > gpurun_out/${T}_plain_nopipe.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_pipe -s 20 -c 1 \
    -o gpurun_out/${T}_pipe $CMD > gpurun_out/${T}_ncu_pipe.log 2>&1
PGTI_SPMM_NOPIPE=1 ncu --set full --clock-control none --import-source on -k regex:k_spmm_win \
    -s 20 -c 1 -o gpurun_out/${T}_win $CMD > gpurun_out/${T}_ncu_win.log 2>&1

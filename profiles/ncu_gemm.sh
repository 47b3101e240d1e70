#!/bin/bash
# ncu --set full of the tcgen05 GEMMs (one of each forward / backward mode) and one staged SpMM
# launch at a workload's shapes (one GPU), after the plain command exits 0.
set -e
CFG=${1:-pems}; T=${2:-gemm}
CMD="python profiles/prof_step.py --config $CFG --steps 1"
$CMD > gpurun_out/${T}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tc_fwd" -s 2 -c 4 \
    -o gpurun_out/${T}_fwd $CMD > gpurun_out/${T}_ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_win" -s 20 -c 1 \
    -o gpurun_out/${T}_spmm $CMD > gpurun_out/${T}_ncu_spmm.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_small_wgrad|k_tc_wgrad|k_tc_reduce|k_small_reduce" -c 12 \
    -o gpurun_out/${T}_wgrad $CMD > gpurun_out/${T}_ncu_wgrad.log 2>&1

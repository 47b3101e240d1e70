#!/bin/bash
# Round-2 ncu --set full evidence at full-PeMS shapes on one B200 (after the plain command exits
# 0): two staged-SpMM launches, the persistent tcgen05 GEMMs (one per mode), the weight-gradient
# kernels and both gather variants.  Summaries: profiles/summarize.py full ...
set -e
CMD="python profiles/prof_step.py --config pems --steps 1"
T=${1:-rd2f}
$CMD > gpurun_out/${T}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_win -s 30 -c 2 \
    -o gpurun_out/${T}_spmm $CMD > gpurun_out/${T}_ncu_spmm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_fwdp -s 2 -c 4 \
    -o gpurun_out/${T}_gemm $CMD > gpurun_out/${T}_ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_small_wgrad|k_tc_wgrad|k_tc_reduce|k_gather|k_cand_bwd_tc" -c 14 \
    -o gpurun_out/${T}_misc $CMD > gpurun_out/${T}_ncu_misc.log 2>&1
PGTI_GATHER=tma $CMD > gpurun_out/${T}_plain_tma.log 2>&1
PGTI_GATHER=tma ncu --set full --clock-control none -k regex:k_gather -c 1 \
    -o gpurun_out/${T}_gather_tma $CMD > gpurun_out/${T}_ncu_tma.log 2>&1

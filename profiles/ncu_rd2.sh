#!/bin/bash
# Round-2 ncu evidence at full-PeMS shapes (one GPU, under gpurun): the plain command first,
# then the launch list of two eager steps and --set full captures of the SpMM, the weight-
# gradient / reduction / elementwise kernels and both gather variants.
set -e
CMD="python profiles/prof_step.py --config ${1:-pems} --steps 2"
T=${2:-rd2}
$CMD > gpurun_out/${T}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_win -s 30 -c 2 \
    -o gpurun_out/${T}_spmm $CMD > gpurun_out/${T}_ncu_spmm.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_small_wgrad|k_small_reduce|k_tc_reduce|k_tc_wgrad|k_cand_bwd_tc|k_gather" -c 16 \
    -o gpurun_out/${T}_misc $CMD > gpurun_out/${T}_ncu_misc.log 2>&1
PGTI_GATHER=tma $CMD > gpurun_out/${T}_plain_tma.log 2>&1
PGTI_GATHER=tma ncu --set full --clock-control none --import-source on -k regex:k_gather -c 1 \
    -o gpurun_out/${T}_gather_tma $CMD > gpurun_out/${T}_ncu_tma.log 2>&1

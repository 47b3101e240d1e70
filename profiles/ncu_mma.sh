#!/bin/bash
# ncu --set full of the tensor-core window SpMM at the full-PeMS shape (after its plain run).
T=${1:-ncu_mma}
export PGTI_SPMM_MMA=1  # (the default at this shape)
CMD="python profiles/prof_step.py --config pems --steps 1"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_mma -s 30 -c 2 \
    -o gpurun_out/${T} $CMD > gpurun_out/${T}_ncu.log 2>&1

#!/bin/bash
# ncu --set full of the tensor-core window SpMM at the METR-LA shape (13 windows, one CTA per SM
# grouping), after its plain run.
CMD="python profiles/prof_step.py --config metr_la --steps 1"
$CMD > gpurun_out/ncu_mma_ml_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_mma -s 30 -c 2 \
    -o gpurun_out/ncu_mma_ml $CMD > gpurun_out/ncu_mma_ml.log 2>&1

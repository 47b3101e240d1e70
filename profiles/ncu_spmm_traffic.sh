#!/bin/bash
# DRAM bytes of EVERY tensor-core SpMM launch of one full-PeMS step (metrics-only ncu pass, after
# the plain command exits 0): the per-launch mean for profiles/traffic_pems.json.
CMD="python profiles/prof_step.py --config pems --steps 1"
$CMD > gpurun_out/spmm_traffic_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_spmm_mma --csv --log-file gpurun_out/spmm_traffic.csv $CMD > gpurun_out/spmm_traffic_ncu.log 2>&1

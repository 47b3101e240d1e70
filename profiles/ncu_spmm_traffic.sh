#!/bin/bash
# DRAM bytes of EVERY SpMM launch of one step of a workload (metrics-only ncu pass, after the
# plain command exits 0): the per-launch mean for profiles/traffic_<config>.json.
C=${1:-pems}
CMD="python profiles/prof_step.py --config $C --steps 1"
$CMD > gpurun_out/spmm_traffic_${C}_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_spmm --csv --log-file gpurun_out/spmm_traffic_${C}.csv $CMD > gpurun_out/spmm_traffic_${C}_ncu.log 2>&1

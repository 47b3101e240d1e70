#!/bin/bash
# DRAM bytes per launch of the SpMM and GEMM kernels of one workload's bench step (ncu, cold
# cache per replayed kernel) -> gpurun_out/traffic_TAG_CONFIG.ncu-rep; run the plain command first.
# Usage: profiles/run_traffic.sh TAG CONFIG [SKIP]
set -e
TAG=$1; CFG=$2; SKIP=${3:-300}
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline --config $CFG"
$CMD > gpurun_out/traffic_plain_${TAG}_$CFG.json 2> gpurun_out/traffic_plain_${TAG}_$CFG.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_spmm|k_tc_fwd|k_tc_wgrad" -s $SKIP -c 12 -o gpurun_out/traffic_${TAG}_$CFG $CMD \
    > gpurun_out/traffic_ncu_${TAG}_$CFG.log 2>&1

#!/bin/bash
# One-call evidence refresh for profiles/ (run under gpurun, single GPU):
#   bench line (default = METR-LA), per-launch device times of one step, ncu --set full of the
#   dominant kernels (SpMM + tcgen05 GEMMs), each only after its plain command exited 0.
# Usage: profiles/refresh.sh TAG [CONFIG]
set -e
TAG=${1:-r03}; CFG=${2:-metr_la}
python bench.py --config $CFG > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
bash profiles/run_launches.sh $TAG "--config $CFG"
CMD="python bench.py --steps 2 --warmup 1 --profile-steps 1 --no-e2e --no-cpu-baseline --config $CFG"
ncu --set full --clock-control none --import-source on -k regex:"k_spmm|k_tc_fwd|k_tc_wgrad" \
    -s 300 -c 8 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1

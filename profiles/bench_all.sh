#!/bin/bash
# Bench lines (every key) for the non-default workloads at HEAD on one B200.
T=${1:-rd2i}
for c in pems_all_la pems_bay metr_la chickenpox; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 300 python bench.py --config metr_la --model encdec --no-cpu-baseline > gpurun_out/${T}_bench_metr_la_encdec.json 2>/dev/null
timeout 300 python bench.py --config metr_la --cheb --no-cpu-baseline > gpurun_out/${T}_bench_metr_la_cheb.json 2>/dev/null

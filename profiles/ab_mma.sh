#!/bin/bash
# A/B of the tensor-core window SpMM (PGTI_SPMM_MMA=1) against the SIMT staged kernels: its
# parity tests first, then bench lines per workload, alternating arms.
T=${1:-ab_mma}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mma or spmm_variants or pipelined" > gpurun_out/${T}_tests.log 2>&1 || exit 1
for c in pems pems_all_la metr_la; do
  for arm in 0 1 0 1; do
    PGTI_SPMM_MMA=$arm timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'mma=$arm', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/${T}_bench.txt
  done
done
PGTI_SPMM_MMA=1 python profiles/prof_step.py --config pems --steps 3 > gpurun_out/${T}_prof.log 2>&1

#!/bin/bash
# r08 evidence at the round's final code: METR-LA bench + launch list + ncu full (SpMM/GEMM),
# bench lines for the other workloads, the oracle arm.  Run under gpurun (1 GPU).
bash profiles/refresh.sh r08 metr_la
for c in pems_bay pems_all_la pems; do
  python bench.py --config $c > gpurun_out/bench_r08_$c.json 2> gpurun_out/bench_r08_$c.err
done
python bench.py --model encdec > gpurun_out/bench_r08_metr_la_encdec.json 2> gpurun_out/bench_r08_encdec.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r08_reference.json 2> gpurun_out/bench_r08_reference.err

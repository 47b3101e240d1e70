#!/bin/bash
# r07 evidence: METR-LA bench + launch list + ncu full (SpMM/GEMM), bench lines for the other
# workloads and variants, a stream timeline.  Run under gpurun (1 GPU).
bash profiles/refresh.sh r07 metr_la
for c in pems_bay pems_all_la pems chickenpox; do
  python bench.py --config $c > gpurun_out/bench_r07_$c.json 2> gpurun_out/bench_r07_$c.err
done
python bench.py --model encdec > gpurun_out/bench_r07_metr_la_encdec.json 2> gpurun_out/bench_r07_encdec.err
python bench.py --cheb > gpurun_out/bench_r07_metr_la_cheb.json 2> gpurun_out/bench_r07_cheb.err
python profiles/timeline.py --json gpurun_out/timeline_r07_metr_la.json > /dev/null 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r07_reference.json 2> gpurun_out/bench_r07_reference.err

#!/bin/bash
# Round-2 confirmation at HEAD on one B200 (b): smoke, the GPU suite, the default bench line (all
# keys), the reference arm, the other workloads, the serialised launch list, and one ncu --set
# full capture of the dominant kernel (the tensor-core window SpMM) after its plain command.
T=${1:-rd2f}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_suite.log 2>&1
S0=$SECONDS; timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
echo "$((SECONDS - S0)) s wall" > gpurun_out/${T}_bench_default.time
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in metr_la pems_bay pems_all_la chickenpox; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 300 python bench.py --config metr_la --model encdec --no-cpu-baseline > gpurun_out/${T}_bench_metr_la_encdec.json 2>/dev/null
bash profiles/launches.sh pems ${T}_pe
CMD="python profiles/prof_step.py --config pems --steps 1"
$CMD > gpurun_out/${T}_ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_mma -s 30 -c 2 \
    -o gpurun_out/${T}_spmm $CMD > gpurun_out/${T}_ncu_spmm.log 2>&1

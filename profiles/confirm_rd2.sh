#!/bin/bash
# Round-2 confirmation at HEAD on one B200: smoke, the GPU suite, the default bench line (all
# keys), the reference arm, METR-LA / PeMS-All-LA / PeMS-Bay lines, the serialised launch list.
T=${1:-rd2}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_suite.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in metr_la pems_bay pems_all_la; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
bash profiles/launches.sh pems ${T}_pe

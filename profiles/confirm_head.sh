#!/bin/bash
# HEAD check on one B200: smoke, the GPU suite, the default bench line.
T=${1:-head}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_suite.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err

timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab12_pems.json 2>/dev/null
timeout 300 python bench.py --config pems_all_la --no-cpu-baseline > gpurun_out/ab12_pal.json 2>/dev/null

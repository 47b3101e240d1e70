timeout 300 python bench.py --config metr_la --no-cpu-baseline > /dev/null 2>&1; cp gpurun_out/kernel_trace_metr_la_n1.json gpurun_out/tr_ml.json
timeout 300 python bench.py --config metr_la --model encdec --no-cpu-baseline > /dev/null 2>&1; cp gpurun_out/kernel_trace_metr_la_n1.json gpurun_out/tr_ed.json
timeout 300 python bench.py --config pems_bay --no-cpu-baseline > /dev/null 2>&1; cp gpurun_out/kernel_trace_pems_bay_n1.json gpurun_out/tr_pb.json

timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mma" > gpurun_out/ab8_tests.log 2>&1
PGTI_SPMM_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mma_oracle or staged or dense_rows" >> gpurun_out/ab8_tests.log 2>&1
bash profiles/ab_env.sh ab8 "pems pems_all_la" - "PGTI_SPMM_PERSIST=1"

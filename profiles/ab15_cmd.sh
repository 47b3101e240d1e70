timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "mma or fragments or staged or dense_rows or bf16" > gpurun_out/ab15_tests.log 2>&1
bash profiles/ab_env.sh ab15 "pems pems_all_la" - "PGTI_SPMM_FRAGS=0"

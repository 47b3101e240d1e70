timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mma or staged or dense_rows" > gpurun_out/ab13_tests.log 2>&1
bash profiles/ab_env.sh ab13 "pems pems_all_la" - "PGTI_SPMM_NST=2"

timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mma" > gpurun_out/ab3_tests.log 2>&1
PGTI_SPMM_NST=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "mma" >> gpurun_out/ab3_tests.log 2>&1
bash profiles/ab_env.sh ab3 "pems pems_all_la" - "PGTI_SPMM_MMA=1" "PGTI_SPMM_MMA=1 PGTI_SPMM_NST=4" "PGTI_SPMM_MMA=1 PGTI_SPMM_NST=2"

timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mma" > gpurun_out/ab5_tests.log 2>&1
bash profiles/ab_env.sh ab5 "pems pems_all_la metr_la" - "PGTI_SPMM_MMA=1" "PGTI_SPMM_MMA=1 PGTI_SPMM_NST=2"

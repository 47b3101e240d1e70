PGTI_SPMM_NST=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "mma" > gpurun_out/ab4_tests.log 2>&1
bash profiles/ab_env.sh ab4 "pems pems_all_la" - "PGTI_SPMM_MMA=1 PGTI_SPMM_NST=2 PGTI_SPMM_BULK=0" "PGTI_SPMM_MMA=1 PGTI_SPMM_NST=2" "PGTI_SPMM_MMA=1 PGTI_SPMM_BULK=0"

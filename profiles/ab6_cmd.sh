timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "mma or spmm_variants or pipelined or staged" > gpurun_out/ab6_tests.log 2>&1
bash profiles/ab_env.sh ab6 "pems pems_all_la" - "PGTI_SPMM_MMA=0" "PGTI_SPMM_NST=2"

timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_trainer.py -q -k "bf16 or tc or fold or fullsize or trainer" > gpurun_out/ab14_tests.log 2>&1
bash profiles/ab_env.sh ab14 "pems pems_all_la metr_la" -

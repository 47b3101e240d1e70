timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bf16 or tc or fold" > gpurun_out/ab11_tests.log 2>&1
bash profiles/ab_env.sh ab11 "pems" -
python profiles/prof_step.py --config pems --steps 1 > /dev/null 2>&1

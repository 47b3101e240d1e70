#!/bin/bash
# Round-2 multi-GPU evidence (run under gpurun --gpus 4): the multi-rank parity tests (2 and 4
# ranks) and the bench at 2 and 4 GPUs (full PeMS with one full epoch at 4, METR-LA), NCCL
# communicator setup logged (NCCL_DEBUG=INFO, INIT) to the .err files.
T=${1:-rd2}
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -s > gpurun_out/${T}_gpu_multi.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --no-e2e \
      $( [ $N = 4 ] && echo --epoch ) > gpurun_out/${T}_bench_pems_n$N.json 2> gpurun_out/${T}_bench_pems_n$N.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29700 + N)) bench.py --gpus $N --config metr_la \
      --no-e2e > gpurun_out/${T}_bench_ml_n$N.json 2> gpurun_out/${T}_bench_ml_n$N.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29800 + N)) bench.py --gpus $N --config pems_all_la \
      --no-e2e > gpurun_out/${T}_bench_pal_n$N.json 2> gpurun_out/${T}_bench_pal_n$N.err
done

#!/bin/bash
# multi-GPU bench lines (torchrun, one rank per GPU): bash profiles/refresh_multi.sh TAG NGPUS
TAG=$1; N=$2
for c in metr_la pems_all_la; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $N --config $c > gpurun_out/bench_${TAG}_${c}_n$N.json \
    2> gpurun_out/bench_${TAG}_${c}_n$N.err
done

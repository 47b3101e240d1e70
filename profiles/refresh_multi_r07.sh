#!/bin/bash
# r07 multi-GPU lines: METR-LA / PeMS-All-LA at N GPUs, plus (N=4) the full-PeMS epoch
N=$1
bash profiles/refresh_multi.sh r07 $N
if [ "$N" = "4" ]; then
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 4 --config pems --epoch --steps 20 \
    > gpurun_out/bench_r07_pems_n4_epoch.json 2> gpurun_out/bench_r07_pems_n4_epoch.err
fi

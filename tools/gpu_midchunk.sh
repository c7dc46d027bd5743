#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3x
for ch in 2048 4096 8192 16384; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$((ch%7)) tools/sweep.py --variants twoshot,oneshot,nccl --mode fast32 --min-kb 256 --max-mb 16 --chunk $ch > gpurun_out/${t}_sweep_ch$ch.log 2>&1
done

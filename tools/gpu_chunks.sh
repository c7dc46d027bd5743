#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3e
i=0
for ch in 65536 262144; do for c in 32 64 0; do
i=$((i+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$i tools/sweep.py --variants twoshot --iters 8 --warmup 2 --min-kb 16384 --ctas $c --chunk $ch > gpurun_out/${t}_ch${ch}_c$c.log 2>&1
done; done

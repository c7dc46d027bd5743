#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3c
for c in 16 32 64 0; do
PGX_TMA=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$((c%10)) tools/sweep.py --variants twoshot --iters 8 --warmup 2 --min-kb 16384 --ctas $c > gpurun_out/${t}_tma_c$c.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$((c%10)) tools/sweep.py --variants twoshot --iters 8 --warmup 2 --min-kb 16384 --ctas $c > gpurun_out/${t}_sm_c$c.log 2>&1
done

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3l
for p in 1 2 4; do
PGX_CE_PARTS=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$p tools/sweep.py --variants twoshot_ce --iters 8 --warmup 2 --min-kb 16384 > gpurun_out/${t}_sweep_p$p.log 2>&1
PGX_CE_PARTS=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$p bench.py --gpus $n --steps 30 --warmup 5 --no-e2e > gpurun_out/${t}_bench_p$p.log 2>&1
done

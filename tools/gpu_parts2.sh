#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3p
for r in 1 2 3; do for p in 1 4; do
PGX_CE_PARTS=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$p bench.py --gpus $n --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${t}_bench_p${p}_r$r.log 2>&1
done; done

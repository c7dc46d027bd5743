#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3q
for r in 1 2; do for g in layer model; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$r bench.py --gpus $n --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --gate $g > gpurun_out/${t}_bench_${g}_r$r.log 2>&1
done; done

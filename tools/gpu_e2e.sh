#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3m
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${t}_bench1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $n > gpurun_out/${t}_bench$n.log 2>&1
timeout 600 python bench.py --workload googlenet --no-cpu-baseline > gpurun_out/${t}_gbench1.log 2>&1

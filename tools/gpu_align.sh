#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r4e
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --variants oneshot_ll,oneshot,twoshot,twoshot_ce,nvls,tree,nccl --mode fast32 > gpurun_out/${t}_sweep_n$n.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29593 tools/sweep.py --variants twoshot,oneshot_ll,nccl --mode sum32 > gpurun_out/${t}_sweep_sum32_n$n.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 tools/sweep.py --variants oneshot_ll,oneshot,twoshot,twoshot_ce,nccl --mode fast32 > gpurun_out/${t}_sweep_n2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29594 bench.py --gpus $n --no-cpu-baseline > gpurun_out/${t}_bench$n.log 2>&1

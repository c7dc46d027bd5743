#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3t
timeout 600 python -m pytest tests/test_gpu_exchange.py -q -x -p no:cacheprovider -rf -k "size_scaled" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --variants twoshot,oneshot,twoshot_ce,twoshot_cep,tree,nvls,nccl --mode fast32 > gpurun_out/${t}_sweep_fast32.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29592 tools/sweep.py --variants twoshot,oneshot,nccl --mode sum32 > gpurun_out/${t}_sweep_sum32.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593 tools/sweep.py --variants twoshot,oneshot,twoshot_ce,nccl --mode fast32 > gpurun_out/${t}_sweep_fast32_n2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${t}_bench1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29594 bench.py --gpus $n > gpurun_out/${t}_bench$n.log 2>&1

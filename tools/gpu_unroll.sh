#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r4d
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "oneshot" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --variants oneshot_ll,oneshot,twoshot,nccl --mode fast32 --max-mb 16 > gpurun_out/${t}_sweep_n$n.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 tools/sweep.py --variants oneshot_ll,oneshot,twoshot,nccl --mode fast32 --max-mb 16 > gpurun_out/${t}_sweep_n2.log 2>&1

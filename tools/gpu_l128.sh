#!/bin/bash
t=r4m
timeout 240 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "l128" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 tools/sweep.py --variants oneshot_l128,oneshot_ll,oneshot,twoshot,nccl --mode fast32 --max-mb 16 --iters 10 --warmup 3 > gpurun_out/${t}_sweep_n2.log 2>&1

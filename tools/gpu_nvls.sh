#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/r1u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1u_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --variants nvls,twoshot,twoshot_ce,nccl --iters 10 --warmup 3 > gpurun_out/r1u_sweep_n$n.log 2>&1
for v in nvls auto; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --variant $v --no-e2e > gpurun_out/r1u_bench_n${n}_$v.log 2>&1
done

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/r1h_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r1h_pytest_multi.log
for v in auto twoshot_ce twoshot nccl_bulk ddp; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --variant $v --no-e2e > gpurun_out/r1h_bench_n${n}_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r1h_bench_n${n}_$v.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --variants twoshot,twoshot_ce,tree,nccl --iters 10 --warmup 3 > gpurun_out/r1h_sweep_n$n.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29536 bench.py --workload googlenet --gpus $n --steps 20 --warmup 5 --variant auto --no-e2e > gpurun_out/r1h_gbench_n$n.log 2>&1

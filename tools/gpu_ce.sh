#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1d_pytest.log
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 tools/sweep.py --variants twoshot,twoshot_ce,nccl --iters 10 --warmup 3 > gpurun_out/r1d_sweep_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/r1d_sweep_n$n.log
for v in twoshot_ce twoshot; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --variant $v > gpurun_out/r1d_bench_n${n}_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r1d_bench_n${n}_$v.log
done
for b in 128 64 32; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --per-gpu-batch $b > gpurun_out/r1d_diag_b$b.log 2>&1
done

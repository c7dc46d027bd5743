#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --variants oneshot,twoshot --iters 10 --warmup 3 --max-mb 16 > gpurun_out/r2b_sweep_n$n.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2b_bench_n${n}_auto.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29536 bench.py --workload googlenet --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2b_gbench_n${n}_auto.log 2>&1

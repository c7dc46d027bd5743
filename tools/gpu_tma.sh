#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/r1r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1r_pytest.log
for t in 1 0; do
PGX_TMA=$t timeout 300 python tools/phase_bench.py --variants twoshot > gpurun_out/r1r_phase_tma$t.log 2>&1
PGX_TMA=$t timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --variants twoshot --iters 10 --warmup 3 > gpurun_out/r1r_sweep_tma$t.log 2>&1
PGX_TMA=$t timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --variant twoshot --no-e2e > gpurun_out/r1r_bench_tma$t.log 2>&1
done

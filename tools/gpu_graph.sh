#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1e_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r1e_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/r1e_bench1.log
n=$(python -c "import torch;print(torch.cuda.device_count())")
for v in twoshot_ce twoshot; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $n --steps 20 --warmup 5 --variant $v > gpurun_out/r1e_bench_n${n}_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r1e_bench_n${n}_$v.log
done
for b in 64 32; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --per-gpu-batch $b > gpurun_out/r1e_diag_b$b.log 2>&1
done

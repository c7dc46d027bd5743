#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/r1i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1i_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --timeline gpurun_out/r1i_timeline_n1_r{rank}.csv > gpurun_out/r1i_bench1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --timeline gpurun_out/r1i_timeline_n${n}_r{rank}.csv > gpurun_out/r1i_bench_n${n}.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus $n --steps 5 --warmup 1 > gpurun_out/r1i_bench_ref_n${n}.log 2>&1

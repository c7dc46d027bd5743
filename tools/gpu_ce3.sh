#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "twoshot_ce or graph" > gpurun_out/r2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --variants twoshot_ce,twoshot --iters 10 --warmup 3 --min-kb 1024 > gpurun_out/r2d_sweep_n$n.log 2>&1
for p in 4 8; do PGX_CE_PARTS=$p timeout 300 python tools/phase_bench.py --variants twoshot_ce > gpurun_out/r2d_phase_p$p.log 2>&1; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r2d_bench_n${n}_auto.log 2>&1

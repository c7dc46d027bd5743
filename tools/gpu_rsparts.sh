#!/bin/bash
# CE per-part push signals (PGX_CE_RS_PARTS) and low-priority large layers, N=4
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3a
PGX_CE_RS_PARTS=1 timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "twoshot_ce or graph or auto" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
for rp in 0 1; do
PGX_CE_RS_PARTS=$rp timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$rp tools/sweep.py --variants twoshot_ce --iters 10 --warmup 3 --min-kb 4096 > gpurun_out/${t}_sweep_rp${rp}.log 2>&1
PGX_CE_RS_PARTS=$rp timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$rp bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${t}_bench_rp${rp}.log 2>&1
done
for pr in 1000000 4000000; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29546 bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --variant twoshot --low-priority-from $pr > gpurun_out/${t}_bench_sm_lp${pr}.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29547 bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --low-priority-from 1000000 > gpurun_out/${t}_bench_auto_lp.log 2>&1

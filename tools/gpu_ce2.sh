#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x -p no:cacheprovider > gpurun_out/r1l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1l_pytest.log
for parts in 1 2 4; do for rs in 1 2; do
PGX_CE_PARTS=$parts PGX_CE_RS_STREAMS=$rs timeout 300 python tools/phase_bench.py --variants twoshot_ce > gpurun_out/r1l_phase_p${parts}_s${rs}.log 2>&1
done; done
for parts in 1 4; do
PGX_CE_PARTS=$parts timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/r1l_bench_n${n}_p${parts}.log 2>&1
done

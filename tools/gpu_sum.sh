#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3n
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x -p no:cacheprovider -rf -k "sum32" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
for ch in 16384 65536; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$((ch%7)) tools/sweep.py --variants twoshot,twoshot_ce,nccl --mode sum32 --chunk $ch > gpurun_out/${t}_sweep_sum32_ch$ch.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29579 tools/sweep.py --variants twoshot,nccl --mode fast32 --chunk 65536 > gpurun_out/${t}_sweep_fast32_ch65536.log 2>&1

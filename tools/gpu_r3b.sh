#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3b
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "after_rendezvous or concurrent" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --steps 30 --warmup 5 --no-e2e > gpurun_out/${t}_bench_n$n.log 2>&1
for b in 64 128; do
timeout 600 python bench.py --per-gpu-batch $b --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${t}_bench1_b$b.log 2>&1
done

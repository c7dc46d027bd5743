#!/bin/bash
# usage: tools/gpu_sweep.sh <tag> ; runs the exchange sweep + AlexNet bench at several CTA caps on all visible GPUs
tag=${1:-sw}
n=$(python -c "import torch;print(torch.cuda.device_count())")
for ctas in ${CTAS_LIST:-0 32 64}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29521 tools/sweep.py --ctas $ctas --iters 10 --warmup 3 > gpurun_out/${tag}_sweep_n${n}_c${ctas}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_sweep_n${n}_c${ctas}.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $n --steps 20 --warmup 5 --max-ctas $ctas --no-e2e > gpurun_out/${tag}_bench_n${n}_c${ctas}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_bench_n${n}_c${ctas}.log
done

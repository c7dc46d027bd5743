#!/bin/bash
# r5w (4 GPUs): TWOSHOT_L128 with finer owner items — parity (1 GPU stepped, 4 GPUs
# concurrent + stress) and the 256 KB - 64 MB sweep at N=2/4.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_benched.py -m gpu -q -x -k "l128 or alexnet or googlenet" > $O/r5w_pytest_l128_1gpu.log 2>&1; echo "stepped rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -q -rA -k "l128 or auto" > $O/r5w_pytest_l128_4gpus.log 2>&1; echo "multi rc=$?"
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
    tools/sweep.py --min-kb 256 --max-mb 64 --variants twoshot_l128,nccl > $O/r5w_sweep_l128_n$n.jsonl 2> $O/r5w_sweep_l128_n$n.err
  echo "sweep n=$n rc=$?"
done
echo done

#!/bin/bash
# r5x (4 GPUs): TWOSHOT_BULK with the copy-engine reduce-scatter (twoshot_ceb): parity
# (stepped 1 GPU, concurrent 4 GPUs), sweep vs the copy-engine and bulk variants, in-step AlexNet.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_exchange.py -m gpu -q -x -k "ceb" > $O/r5x_pytest_ceb_1gpu.log 2>&1; echo "stepped rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -rA -k "ceb" > $O/r5x_pytest_ceb_4gpus.log 2>&1; echo "multi rc=$?"
for c in 24 48; do
  timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 297$c \
    tools/sweep.py --min-kb 16384 --max-mb 256 --ctas $c --variants twoshot_ceb,twoshot_bulk > $O/r5x_sweep_n4_c$c.jsonl 2> $O/r5x_sweep_n4_c$c.err
  echo "sweep c=$c rc=$?"
done
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29851 $B > $O/r5x_bench4_ce.json 2> $O/r5x_bench4_ce.err; echo "b0 rc=$?"
timeout 900 $TR --master-port 29852 $B --large ceb --large-ctas 24 > $O/r5x_bench4_ceb24.json 2> $O/r5x_bench4_ceb24.err; echo "b1 rc=$?"
timeout 900 $TR --master-port 29853 $B --large ceb --large-ctas 48 > $O/r5x_bench4_ceb48.json 2> $O/r5x_bench4_ceb48.err; echo "b2 rc=$?"
timeout 900 $TR --master-port 29854 $B --large ceb --large-ctas 24 --xflags bulk_lean > $O/r5x_bench4_ceb24_lean.json 2> $O/r5x_bench4_ceb24_lean.err; echo "b3 rc=$?"
timeout 900 $TR --master-port 29855 $B --large ceb --large-ctas 48 --xflags bulk_lean > $O/r5x_bench4_ceb48_lean.json 2> $O/r5x_bench4_ceb48_lean.err; echo "b4 rc=$?"
timeout 900 $TR --master-port 29856 $B > $O/r5x_bench4_ce_b.json 2> $O/r5x_bench4_ce_b.err; echo "b5 rc=$?"
echo done

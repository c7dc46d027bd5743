#!/bin/bash
# r5s (4 GPUs): TWOSHOT_L128 first light — stepped parity on one GPU, concurrent parity on
# 2/4 GPUs, 1-16 MB sweeps at N=2/4 against the existing variants and NCCL; ref64 sweep row;
# in-step AlexNet N=4 with lean bulk CTA caps.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_exchange.py -m gpu -q -rA -k "l128" -x > $O/r5s_pytest_l128_1gpu.log 2>&1
echo "stepped rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -q -rA -k "l128" > $O/r5s_pytest_l128_4gpus.log 2>&1
echo "multi rc=$?"
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n \
    tools/sweep.py --min-kb 256 --max-mb 16 --variants twoshot_l128,oneshot_l128,twoshot,oneshot,oneshot_ll,nccl \
    > $O/r5s_sweep_mid_n$n.jsonl 2> $O/r5s_sweep_mid_n$n.err
  echo "sweep n=$n rc=$?"
done
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29911 tools/sweep.py --mode ref64 \
  --min-kb 4 --max-mb 64 --variants twoshot,tree,oneshot,nccl > $O/r5s_sweep_ref64_n4.jsonl 2> $O/r5s_sweep_ref64.err
echo "ref64 rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29921 $B > $O/r5s_bench4_ce.json 2> $O/r5s_bench4_ce.err
for c in 16 24 32; do
  timeout 900 $TR --master-port 2993$c $B --large bulk --large-ctas $c --xflags bulk_lean > $O/r5s_bench4_bulk${c}_lean.json 2> $O/r5s_bench4_bulk${c}_lean.err
done
timeout 900 $TR --master-port 29941 $B --large bulk --large-ctas 24 > $O/r5s_bench4_bulk24.json 2> $O/r5s_bench4_bulk24.err
echo done

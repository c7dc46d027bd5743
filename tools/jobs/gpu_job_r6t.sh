#!/bin/bash
# r6t (2 GPUs): PGX_XF_LEAN_CAPPED (128-thread CTAs for the capped LL / L128 layers):
# GoogLeNet plan parity with it (1 GPU stepped), GoogLeNet and AlexNet N=2 with/without.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6t
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_benched.py -m gpu -x -q -k "googlenet" > $O/${R}_pytest.log 2>&1; echo "test rc=$?"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 600 $TR2 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b g_def --workload googlenet
b g_lean --workload googlenet --xflags lean_capped
b g_defb --workload googlenet
b g_leanb --workload googlenet --xflags lean_capped
b a_def
b a_lean --xflags lean_capped
echo done

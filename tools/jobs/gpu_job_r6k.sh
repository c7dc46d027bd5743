#!/bin/bash
# r6k (4 GPUs): overlap_ctas — the small layers hidden behind the backward on capped grids,
# layer 0 (the exposed one) on the full grid: parity (GoogLeNet plans, 1 GPU stepped) and
# in-step GoogLeNet N=4 / AlexNet N=4 and N=2, alternating with the uncapped default.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6k
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_benched.py -m gpu -x -q -k "googlenet" > $O/${R}_pytest_1gpu.log 2>&1; echo "suite1 rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
B2="bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_bench4_$name.json 2> $O/${R}_bench4_$name.err; echo "$name rc=$?"; }
b2() { local name=$1; shift; p=$((p+1)); timeout 900 $TR2 --master-port $p $B2 "$@" > $O/${R}_bench2_$name.json 2> $O/${R}_bench2_$name.err; echo "$name rc=$?"; }
b g_def --workload googlenet
b g_ov16 --workload googlenet --overlap-ctas 16
b g_ov8 --workload googlenet --overlap-ctas 8
b g_ov16b --workload googlenet --overlap-ctas 16
b g_defb --workload googlenet
b a_def
b a_ov16 --overlap-ctas 16
b a_ov8 --overlap-ctas 8
b a_defb
b a_ov16b --overlap-ctas 16
b2 a_def
b2 a_ov16 --overlap-ctas 16
echo done

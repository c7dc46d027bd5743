#!/bin/bash
# r6i (4 GPUs): GoogLeNet step vs its compute (N=1 at B=32 = fwd+bwd + a 7 M-param update),
# gate layer vs model at N=4; AlexNet NCCL comparison rows (DDP, bulk-synchronous NCCL) on
# the current build at N=4 and N=2; AlexNet N=2 with the TMA bulk kernel at 48 CTAs.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6i
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --workload googlenet --per-gpu-batch 32 --no-cpu-baseline --steps 30 > $O/${R}_gbench1_b32.json 2> $O/${R}_gbench1_b32.err; echo "g1 rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
B2="bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_bench4_$name.json 2> $O/${R}_bench4_$name.err; echo "$name rc=$?"; }
b2() { local name=$1; shift; p=$((p+1)); timeout 900 $TR2 --master-port $p $B2 "$@" > $O/${R}_bench2_$name.json 2> $O/${R}_bench2_$name.err; echo "$name rc=$?"; }
b g_model --workload googlenet
b g_layer --workload googlenet --gate layer
b ce
b ddp --variant ddp
b nccl_bulk --variant nccl_bulk
b2 ce
b2 bulk48 --large bulk --large-ctas 48
b2 ddp --variant ddp
echo done

#!/bin/bash
# r6n (4 GPUs): GoogLeNet N=4 --overlap-exposed sweep (r6m: 5 gave 9.31 ms vs 9.62 for 1 and
# 9.66-9.68 for 2/3): 4, 5, 6, 8, 12 and repeats; AlexNet with 5 (= every conv layer full).
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6n
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b g_e5 --workload googlenet --overlap-exposed 5
b g_e4 --workload googlenet --overlap-exposed 4
b g_e6 --workload googlenet --overlap-exposed 6
b g_e8 --workload googlenet --overlap-exposed 8
b g_e12 --workload googlenet --overlap-exposed 12
b g_e1 --workload googlenet
b g_e5b --workload googlenet --overlap-exposed 5
b g_e0 --workload googlenet --overlap-ctas 0
b g_e5_layer --workload googlenet --overlap-exposed 5 --gate layer
b a_e5 --overlap-exposed 5
echo done

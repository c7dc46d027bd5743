#!/bin/bash
# r6m (4 GPUs): how many of the last-emitted layers should keep the full grid
# (--overlap-exposed 1/2/3/5), GoogLeNet N=4 and AlexNet N=4, alternating.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6m
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b g_e1 --workload googlenet
b g_e2 --workload googlenet --overlap-exposed 2
b g_e3 --workload googlenet --overlap-exposed 3
b g_e5 --workload googlenet --overlap-exposed 5
b g_e3_layer --workload googlenet --overlap-exposed 3 --gate layer
b g_e1b --workload googlenet
b g_e3b --workload googlenet --overlap-exposed 3
b a_e1
b a_e2 --overlap-exposed 2
b a_e1b
b a_e2b --overlap-exposed 2
echo done

#!/bin/bash
# r6j (4 GPUs): GoogLeNet N=4 (9.82 ms/step vs 9.36 ms at N=1, B=32): the small layers'
# exchange launches with capped grids (fewer SMs taken from the backward), at normal stream
# priority, and without the L128 band.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6j
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline --workload googlenet"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_gbench4_$name.json 2> $O/${R}_gbench4_$name.err; echo "$name rc=$?"; }
b def_a
b cap16 --max-ctas 16
b cap32 --max-ctas 32
b cap64 --max-ctas 64
b lowprio --low-priority-from 1
b nol128 --l128 ''
b cap8 --max-ctas 8
b def_b
b cap32_lp --max-ctas 32 --low-priority-from 1
echo done

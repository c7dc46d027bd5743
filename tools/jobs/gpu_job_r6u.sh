#!/bin/bash
# r6u (2 GPUs): GoogLeNet / AlexNet N=2 with every exchange stream at normal priority
# (--low-priority-from 1) next to the default high-priority stream, with the 16-CTA caps.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6u
mkdir -p $O
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 600 $TR2 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b g_def --workload googlenet
b g_lp --workload googlenet --low-priority-from 1
b g_defb --workload googlenet
b g_lpb --workload googlenet --low-priority-from 1
b a_def
b a_lp --low-priority-from 1
echo done

#!/bin/bash
# r6v (2 GPUs): the step graph instantiated with node priorities (--graph-prio) vs torch's
# instantiation; GoogLeNet N=2 steps are bimodal (9.26 / 9.60-9.64 ms, r6u).
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6v
mkdir -p $O
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 600 $TR2 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b g_prio --workload googlenet --graph-prio
b g_def --workload googlenet
b g_prio2 --workload googlenet --graph-prio
b g_defb --workload googlenet
b g_prio3 --workload googlenet --graph-prio
b a_prio --graph-prio
b a_def
echo done

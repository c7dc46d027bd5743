#!/bin/bash
# r6p (4 GPUs): comparison rows in the AlexNet N=4 step — every layer on the paper's tree
# schedule, every layer on NVLS (switch-side reduce, fp32 tolerance parity), every layer on
# the SM two-shot — beside the default plan.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6p
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b auto
b tree --variant tree
b nvls --variant nvls
b twoshot --variant twoshot
b auto_b
echo done

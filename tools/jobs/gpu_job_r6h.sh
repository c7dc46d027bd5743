#!/bin/bash
# r6h (4 GPUs): where the N=4 step's ~0.1 ms over compute goes: fwd+bwd alone (no optimizer)
# at B=256/128/64, traced timelines (CSV per rank) for ce and bulk 48, exchange streams at
# normal priority for the large layers (--low-priority-from 1M) vs the default high priority.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6h
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 OPT=none FAST=1 BATCHES=256,128,64 timeout 600 python tools/fwdbwd_variants.py > $O/${R}_fwdbwd_none.log 2>&1; echo "fwdbwd rc=$?"
CUDA_VISIBLE_DEVICES=0 OPT=sgd FAST=1 BATCHES=128 timeout 600 python tools/fwdbwd_variants.py > $O/${R}_fwdbwd_sgd.log 2>&1; echo "fwdbwd rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_bench4_$name.json 2> $O/${R}_bench4_$name.err; echo "$name rc=$?"; }
b ce_tl --timeline $O/${R}_tl_ce_r{rank}.csv
b bulk48_tl --large bulk --large-ctas 48 --timeline $O/${R}_tl_bulk48_r{rank}.csv
b ce_lp --low-priority-from 1048576
b bulk48_lp --large bulk --large-ctas 48 --low-priority-from 1048576
b cet64_lp --large cet --large-ctas 64 --low-priority-from 1048576
b ce_a
b bulk48_lp2 --large bulk --large-ctas 48 --low-priority-from 1048576
b ce_b
echo done

#!/bin/bash
# r6d (4 GPUs): in-step AlexNet N=4, alternating order on one box: ce (default) vs cet
# (copy engines + TMA-fed owner fold) at 64/96 CTAs vs ceb (copy-engine reduce-scatter +
# TMA owner + TMA all-gather) at 32/64 CTAs; N=4 sweep of ceb; GoogLeNet N=4 ce vs cet64.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6d
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_bench4_$name.json 2> $O/${R}_bench4_$name.err; echo "$name rc=$?"; }
b ce_a
b cet64_a --large cet --large-ctas 64
b ceb32_a --large ceb --large-ctas 32
b cet96_a --large cet --large-ctas 96
b ce_b
b cet64_b --large cet --large-ctas 64
b ceb64_a --large ceb --large-ctas 64
b ce_c
b cet64_c --large cet --large-ctas 64
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/sweep.py --min-kb 16384 --max-mb 256 \
  --ctas 32 --variants twoshot_ceb > $O/${R}_sweep_n4_ceb32.jsonl 2> $O/${R}_sweep_n4_ceb32.err; echo "sweep rc=$?"
b g_ce --workload googlenet
b g_cet64 --workload googlenet --large cet --large-ctas 64
echo done

#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5p: N=4 in-step: CE vs bulk full / lean footprints.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29811 tools/sweep.py --min-kb 4096 --max-mb 256 --variants twoshot_bulk --ctas 48 > $O/r5p_sweep_n4_bulk48_full.jsonl 2> $O/r5p_sweep.err
timeout 300 $TR --master-port 29817 tools/sweep.py --min-kb 4096 --max-mb 256 --variants twoshot_bulk --ctas 48 --xflags bulk_lean > $O/r5p_sweep_n4_bulk48_lean.jsonl 2>> $O/r5p_sweep.err
timeout 300 $TR --master-port 29812 tools/nvlink_counters.py --mb 144 --variants twoshot,twoshot_ce,nccl --reps 20 > $O/r5p_nvlink_n4.jsonl 2> $O/r5p_nvlink.err
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29813 $B > $O/r5p_bench4_ce.json 2> $O/r5p_bench4_ce.err
timeout 900 $TR --master-port 29814 $B --large bulk --large-ctas 48 > $O/r5p_bench4_bulk48.json 2> $O/r5p_bench4_bulk48.err
timeout 900 $TR --master-port 29815 $B --large bulk --large-ctas 48 --xflags bulk_lean > $O/r5p_bench4_bulk48_lean.json 2> $O/r5p_bench4_bulk48_lean.err
timeout 900 $TR --master-port 29816 $B --large bulk --large-ctas 96 --xflags bulk_lean > $O/r5p_bench4_bulk96_lean.json 2> $O/r5p_bench4_bulk96_lean.err
echo done

#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5l: bulk owner A/B (store lag, LSU local stores), N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
L=paper_1706_00095_b200
cp $L/libpgx.so $L/libpgx_v_base.so
P=29720
for v in base lag3 stg stg_lag3; do
  P=$((P+1))
  cp $L/libpgx_v_$v.so $L/libpgx.so
  timeout 300 $TR --master-port $P tools/trace_oneshot.py --variant twoshot_bulk --kb 65536 > $O/r5l_trace_$v.jsonl 2> $O/r5l_trace_$v.err
  P=$((P+1))
  timeout 300 $TR --master-port $P tools/sweep.py --min-kb 65536 --max-mb 256 --variants twoshot_bulk --ctas 32 > $O/r5l_sweep_$v.jsonl 2> $O/r5l_sweep_$v.err
done

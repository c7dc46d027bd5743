#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5g: bulk owner-loop accumulators, N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
P=29660
for c in 24; do
  P=$((P+1))
  timeout 300 $TR --master-port $P tools/trace_oneshot.py --variant twoshot_bulk --kb 65536 --ctas $c > $O/r5g_trace_bulk_64mb_c$c.jsonl 2> $O/r5g_trace_bulk_c$c.err
done
timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -k "twoshot_bulk" > $O/r5g_pytest_bulk.log 2>&1
echo "bulk stepped rc=$?"

#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5m: LSU-fold bulk owner, N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -k "twoshot_bulk" > $O/r5m_pytest_bulk.log 2>&1
echo "bulk stepped rc=$?"
timeout 300 $TR --master-port 29740 tools/trace_oneshot.py --variant twoshot_bulk --kb 65536 > $O/r5m_trace_bulk_64mb_c24.jsonl 2> $O/r5m_trace.err
P=29741
for c in 16 24 32 48; do
  P=$((P+1))
  timeout 300 $TR --master-port $P tools/sweep.py --min-kb 4096 --max-mb 256 --variants twoshot_bulk --ctas $c > $O/r5m_sweep_n2_bulk_c$c.jsonl 2> $O/r5m_sweep_n2_bulk_c$c.err
done

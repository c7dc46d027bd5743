#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5c: bulk CTA sweep, stress, N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
P=29600
for c in 16 32 48; do
  P=$((P+1))
  timeout 300 $TR --master-port $P tools/sweep.py --min-kb 4096 --variants twoshot_bulk --ctas $c > $O/r5c_sweep_n2_bulk_c$c.jsonl 2> $O/r5c_sweep_n2_bulk_c$c.err
done
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_checkpoint.py -x -q > $O/r5c_pytest_stress.log 2>&1
echo "stress rc=$?"

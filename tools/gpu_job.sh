#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5i: bulk owner fence placement A/B, N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29680 tools/trace_oneshot.py --variant twoshot_bulk --kb 65536 > $O/r5i_trace_fence_all.jsonl 2> $O/r5i_trace.err
cp paper_1706_00095_b200/libpgx_fence_t0.so paper_1706_00095_b200/libpgx.so
timeout 300 $TR --master-port 29681 tools/trace_oneshot.py --variant twoshot_bulk --kb 65536 > $O/r5i_trace_fence_t0.jsonl 2>> $O/r5i_trace.err

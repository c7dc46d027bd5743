#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5n: N=4 sweep, NVLink counters, in-step benches.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29801 tools/sweep.py --min-kb 1024 --max-mb 256 --variants twoshot,twoshot_ce,twoshot_bulk,nccl > $O/r5n_sweep_n4.jsonl 2> $O/r5n_sweep_n4.err
echo "sweep rc=$?"
timeout 300 $TR --master-port 29802 tools/sweep.py --min-kb 4096 --max-mb 256 --variants twoshot_bulk --ctas 48 > $O/r5n_sweep_n4_bulk_c48.jsonl 2> $O/r5n_sweep_n4_bulk_c48.err
timeout 300 $TR --master-port 29803 tools/nvlink_counters.py --mb 144 --variants twoshot,twoshot_bulk,twoshot_ce,nccl > $O/r5n_nvlink_n4.jsonl 2> $O/r5n_nvlink_n4.err
echo "nvlink rc=$?"
timeout 900 $TR --master-port 29804 bench.py --gpus 4 --steps 30 --warmup 5 > $O/r5n_bench4_ce.json 2> $O/r5n_bench4_ce.err
echo "bench ce rc=$?"
timeout 900 $TR --master-port 29805 bench.py --gpus 4 --steps 30 --warmup 5 --large bulk --no-cpu-baseline > $O/r5n_bench4_bulk.json 2> $O/r5n_bench4_bulk.err
timeout 900 $TR --master-port 29806 bench.py --gpus 4 --steps 30 --warmup 5 --large bulk --large-ctas 48 --no-cpu-baseline > $O/r5n_bench4_bulk48.json 2> $O/r5n_bench4_bulk48.err
echo "bench bulk rc=$?"

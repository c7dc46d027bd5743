#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5a: bulk two-shot first light at N=2.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
TR="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
nvidia-smi topo -m > $O/r5a_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange.py -x -q -k "twoshot_bulk" > $O/r5a_pytest_bulk.log 2>&1
echo "bulk stepped rc=$?"
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "twoshot_bulk" > $O/r5a_pytest_multi_bulk.log 2>&1
echo "bulk multi rc=$?"
timeout 600 $TR --master-port 29511 tools/sweep.py --min-kb 1024 --variants twoshot,twoshot_ce,twoshot_bulk,nccl > $O/r5a_sweep_n2.jsonl 2> $O/r5a_sweep_n2.err
echo "sweep rc=$?"
for c in 16 32 48; do
  timeout 300 $TR --master-port 2952$c tools/sweep.py --min-kb 4096 --variants twoshot_bulk --ctas $c > $O/r5a_sweep_n2_bulk_c$c.jsonl 2> $O/r5a_sweep_n2_bulk_c$c.err
done
timeout 600 $TR --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/r5a_bench2_ce.json 2> $O/r5a_bench2_ce.err
echo "bench ce rc=$?"
timeout 600 $TR --master-port 29532 bench.py --gpus 2 --steps 20 --warmup 5 --large bulk --no-cpu-baseline > $O/r5a_bench2_bulk.json 2> $O/r5a_bench2_bulk.err
echo "bench bulk rc=$?"
timeout 1500 python -m pytest tests/test_gpu_benched.py -x -q > $O/r5a_pytest_benched.log 2>&1
echo "benched rc=$?"

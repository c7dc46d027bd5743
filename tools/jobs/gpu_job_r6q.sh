#!/bin/bash
# r6q (4 GPUs): benched-plan parity after the layer_ctas refactor (1 GPU), then the
# copy-engine owner pipelining depth in the step (--ce-parts 2/3/4/6) at N=4 and N=2.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6q
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_benched.py -m gpu -x -q > $O/${R}_pytest_benched_1gpu.log 2>&1; echo "benched rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b2() { local name=$1; shift; p=$((p+1)); timeout 900 $TR2 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
b p4
b p2 --ce-parts 2
b p3 --ce-parts 3
b p6 --ce-parts 6
b p4b
b p2b --ce-parts 2
b2 n2_p4
b2 n2_p2 --ce-parts 2
b2 n2_p6 --ce-parts 6
echo done

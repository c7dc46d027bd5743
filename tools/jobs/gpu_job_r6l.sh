#!/bin/bash
# r6l (4 GPUs): the round-2 final build across real GPUs — the multi-GPU + stress suite,
# then bench lines with the final defaults: AlexNet N=4 (x2) / N=2, GoogLeNet N=4 (model and
# layer gates), configs[0] LeNet 2-rank and configs[1] cifar10_quick 4-rank with their
# reference arms, AlexNet N=4 with --large cet.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6l
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -q > $O/${R}_pytest_multi_4gpus.log 2>&1; echo "multi rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
p=29900
r4() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
r2() { local name=$1; shift; p=$((p+1)); timeout 900 $TR2 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 "$@" > $O/${R}_$name.json 2> $O/${R}_$name.err; echo "$name rc=$?"; }
r4 bench4 --no-cpu-baseline
r4 bench4b --no-cpu-baseline
r4 bench4_cet64 --no-cpu-baseline --large cet --large-ctas 64
r2 bench2 --no-cpu-baseline
r4 gbench4 --no-cpu-baseline --workload googlenet
r4 gbench4_layer --no-cpu-baseline --workload googlenet --gate layer
r2 lenet2 --workload lenet
r2 lenet2_ref --workload lenet --impl reference
r4 cifar4 --workload cifar10_quick
r4 cifar4_ref --workload cifar10_quick --impl reference
echo done

#!/bin/bash
# r6r (2 GPUs): the fwd_bwd_alone field of the bench line (forward + backward with the
# exchange switched off, same process) at N=1 and N=2; GoogLeNet N=2.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6r
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-cpu-baseline > $O/${R}_bench1.json 2> $O/${R}_bench1.err; echo "b1 rc=$?"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29901 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline > $O/${R}_bench2.json 2> $O/${R}_bench2.err; echo "b2 rc=$?"
timeout 900 $TR2 --master-port 29902 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --workload googlenet > $O/${R}_gbench2.json 2> $O/${R}_gbench2.err; echo "g2 rc=$?"
echo done

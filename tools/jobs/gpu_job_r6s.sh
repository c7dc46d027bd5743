#!/bin/bash
# r6s (2 GPUs): graph-mode per-layer exchange spans (--trace-graph) for AlexNet and GoogLeNet
# at N=2; the ModuleBinding.disabled GPU test.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6s
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_gpu_exchange.py -m gpu -q -k "module_binding" > $O/${R}_pytest.log 2>&1; echo "test rc=$?"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29901 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --trace-graph > $O/${R}_bench2.json 2> $O/${R}_bench2.err; echo "b2 rc=$?"
timeout 900 $TR2 --master-port 29902 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --trace-graph --workload googlenet > $O/${R}_gbench2.json 2> $O/${R}_gbench2.err; echo "g2 rc=$?"
echo done

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3f
run() { name=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --no-e2e "$@" > gpurun_out/${t}_$name.log 2>&1; }
run auto
run sm_ch64k_c32 --variant twoshot --chunk-elems 65536 --max-ctas 32
run sm_ch64k_c64 --variant twoshot --chunk-elems 65536 --max-ctas 64
run sm_ch64k_c0 --variant twoshot --chunk-elems 65536
run sm_ch64k_c32_lp --variant twoshot --chunk-elems 65536 --max-ctas 32 --low-priority-from 1000000

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3g
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "concurrent or auto or graph" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
run() { name=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --no-e2e "$@" > gpurun_out/${t}_$name.log 2>&1; }
run ce
for c in 48 64 96; do for ch in 65536 131072; do
run sm_c${c}_ch${ch} --large sm --large-ctas $c --large-chunk-elems $ch
done; done
run sm_c0_ch65536 --large sm --large-chunk-elems 65536

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3w
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "real_models or dead_peer" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
for r in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$r bench.py --gpus $n --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${t}_bench${n}_r$r.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-e2e --no-cpu-baseline > gpurun_out/${t}_bench2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --workload googlenet --no-e2e --no-cpu-baseline > gpurun_out/${t}_gbench$n.log 2>&1

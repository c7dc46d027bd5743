#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r4j
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "oneshot or graph" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --variants oneshot,nccl --mode fast32 --min-kb 256 --max-mb 4 > gpurun_out/${t}_sweep_n$n.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29597 tools/trace_oneshot.py --kb 1024 > gpurun_out/${t}_trace.log 2>&1

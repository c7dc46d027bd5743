#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3r
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "tree or nvls or size_scaled" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
for a in 0 1; do
PGX_AUTO_CHUNK_TREE=$a PGX_AUTO_CHUNK_NVLS=$a timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$a tools/sweep.py --variants tree,nvls --mode fast32 --min-kb 1024 > gpurun_out/${t}_sweep_auto$a.log 2>&1
done

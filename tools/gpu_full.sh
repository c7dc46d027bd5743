#!/bin/bash
# usage: tools/gpu_full.sh <tag> : full GPU test suite + bench on all visible GPUs for each variant
tag=${1:-full}
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench1.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_bench1.log
n=$(python -c "import torch;print(torch.cuda.device_count())")
if [[ $n -ge 2 ]]; then
for v in ${VARIANTS:-twoshot_ce twoshot tree}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $n --steps 20 --warmup 5 --variant $v > gpurun_out/${tag}_bench_n${n}_$v.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_bench_n${n}_$v.log
done
fi

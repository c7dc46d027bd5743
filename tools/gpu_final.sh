#!/bin/bash
# full GPU suite + AlexNet bench for each policy on all visible GPUs, plus N=1
tag=${1:-fin}
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench1.log 2>&1
for v in ${VARIANTS:-auto twoshot twoshot_ce}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $n --steps 20 --warmup 5 --variant $v > gpurun_out/${tag}_bench_n${n}_$v.log 2>&1
done

#!/bin/bash
# round-end numbers: full GPU suite, AlexNet N=1 (+CPU baseline), N=2, N=4, GoogLeNet N=1/4, reference arm
tag=${1:-fin}
n=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench1.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench1_ref.log 2>&1
timeout 600 python bench.py --workload googlenet --no-cpu-baseline > gpurun_out/${tag}_gbench1.log 2>&1
for k in 2 $n; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 --master-port 2954$k bench.py --gpus $k > gpurun_out/${tag}_bench$k.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29549 bench.py --workload googlenet --gpus $n > gpurun_out/${tag}_gbench$n.log 2>&1

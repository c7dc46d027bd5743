#!/bin/bash
# usage: tools/gpu_run.sh <tag> [pytest|bench1|bench2|all]
tag=${1:-run}; what=${2:-all}
mkdir -p gpurun_out
if [[ $what == all || $what == pytest ]]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
if [[ $what == all || $what == bench1 ]]; then
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench1.log 2>&1
  echo "bench1 rc=$?" >> gpurun_out/${tag}_bench1.log
fi
if [[ $what == all || $what == bench2 ]]; then
  n=$(python -c "import torch;print(torch.cuda.device_count())")
  if [[ $n -ge 2 ]]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/${tag}_bench${n}.log 2>&1
    echo "bench$n rc=$?" >> gpurun_out/${tag}_bench${n}.log
  fi
fi

#!/bin/bash
n=$(python -c "import torch;print(torch.cuda.device_count())")
t=r3i
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_multi.py -q -x -p no:cacheprovider -rf -k "cep" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/sweep.py --variants twoshot_cep,twoshot_ce --iters 8 --warmup 2 --min-kb 4096 --chunk 65536 > gpurun_out/${t}_sweep.log 2>&1
run() { name=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 5 --no-e2e "$@" > gpurun_out/${t}_$name.log 2>&1; }
run ce
run cep_ch64k --large cep --large-chunk-elems 65536
run cep_ch64k_c32 --large cep --large-chunk-elems 65536 --large-ctas 32
run cep_ch64k_c96 --large cep --large-chunk-elems 65536 --large-ctas 96
run cep_ch16k --large cep

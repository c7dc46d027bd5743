#!/bin/bash
t=r3j
timeout 600 python -m pytest tests/test_gpu_checkpoint.py -q -x -p no:cacheprovider -rf > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log
timeout 300 python tools/ckpt_bench.py > gpurun_out/${t}_ckpt_bench.json 2> gpurun_out/${t}_ckpt_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_smoke.log

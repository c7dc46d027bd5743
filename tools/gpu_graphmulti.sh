#!/bin/bash
t=r4a
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_exchange.py -q -p no:cacheprovider -rf -k "graph" > gpurun_out/${t}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${t}_pytest.log

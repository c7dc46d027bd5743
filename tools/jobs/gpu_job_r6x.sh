#!/bin/bash
# r6x (1 GPU): the graph-helper and ModuleBinding tests added last.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_exchange.py -m gpu -q -k "graph or module_binding" > $O/r6x_pytest.log 2>&1; echo "rc=$?"

#!/bin/bash
# r6y (1 GPU): N=1 bench of the submitted tree (after the bench.py cleanup) + smoke.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r6y_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --no-cpu-baseline > $O/r6y_bench1.json 2> $O/r6y_bench1.err; echo "bench rc=$?"

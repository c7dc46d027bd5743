#!/bin/bash
# Final 1-GPU rehearsal (what the driver runs at round end): full -m gpu suite, smoke,
# bench N=1 default line, reference arm.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=${R:-r6w}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${R}_pytest_gpu_1gpu.log 2>&1; echo "suite rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/${R}_bench1.json 2> $O/${R}_bench1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_bench1_ref.json 2> $O/${R}_bench1_ref.err; echo "ref rc=$?"
echo done

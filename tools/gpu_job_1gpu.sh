#!/bin/bash
# r6f (1 GPU): driver rehearsal on the round-2 build (full -m gpu suite, smoke, N=1 bench +
# reference arm), N=1 fused-update chunk/CTA sweep (tools/prof_update.py), compute-only
# AlexNet fwd+bwd at B=256/64/32 (tools/fwdbwd_variants.py).
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
R=${R:-r6f}
mkdir -p $O
timeout 600 python tools/prof_update.py 16384:0 4096:0 8192:0 32768:0 65536:0 16384:296 8192:296 4096:296 2048:0 > $O/${R}_prof_update.jsonl 2> $O/${R}_prof_update.err; echo "prof rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${R}_pytest_gpu_1gpu.log 2>&1; echo "suite rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/${R}_bench1.json 2> $O/${R}_bench1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/${R}_bench1_ref.json 2> $O/${R}_bench1_ref.err; echo "ref rc=$?"
timeout 600 python tools/fwdbwd_variants.py > $O/${R}_fwdbwd.log 2>&1; echo "fwdbwd rc=$?"
echo done

#!/bin/bash
# r6o (1 GPU): final rehearsal of the round-2 build: N=1 update sweep, full -m gpu suite + smoke,
# suite + smoke, N=1 bench x2, the bench's launch list (ncu gpu__time_duration) and an
# ncu --set full capture of the fc6 update (traffic for roofline.traffic).
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=${R:-r6o}
mkdir -p $O
timeout 600 python tools/prof_update.py 16384:0 16384:296 > $O/${R}_prof_update.jsonl 2> $O/${R}_prof_update.err; echo "prof rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${R}_pytest_gpu_1gpu.log 2>&1; echo "suite rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/${R}_bench1.json 2> $O/${R}_bench1.err; echo "bench rc=$?"
timeout 900 python bench.py > $O/${R}_bench1b.json 2> $O/${R}_bench1b.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/${R}_launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${R}_launches_n1.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_twoshot -s 5 -c 3 -o $O/${R}_ncu_update \
  python tools/prof_update.py 16384:0 > $O/${R}_ncu_update.log 2>&1; echo "ncu rc=$?"
ncu -i $O/${R}_ncu_update.ncu-rep --page raw --csv > $O/${R}_ncu_update_raw.csv 2>/dev/null
ncu -i $O/${R}_ncu_update.ncu-rep --page details --csv > $O/${R}_ncu_update_details.csv 2>/dev/null
rm -f $O/${R}_ncu_update.ncu-rep
echo done

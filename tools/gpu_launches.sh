#!/bin/bash
t=r4c
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${t}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${t}_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${t}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${t}_ncu.log

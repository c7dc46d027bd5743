#!/bin/bash
t=r4h
timeout 300 python tools/ckpt_bench.py > gpurun_out/${t}_plain.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ckpt -c 2 -o gpurun_out/${t}_ckpt python tools/ckpt_bench.py > gpurun_out/${t}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${t}_ncu.log

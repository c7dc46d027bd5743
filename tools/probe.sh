#!/bin/bash
nvidia-smi > gpurun_out/probe_smi.txt 2>&1
nvidia-smi topo -m >> gpurun_out/probe_smi.txt 2>&1
nproc >> gpurun_out/probe_smi.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/probe_smi.txt
python - >> gpurun_out/probe_smi.txt 2>&1 <<'PY'
import torch, os
print("devices", torch.cuda.device_count(), os.sched_getaffinity(0).__len__())
n = torch.cuda.device_count()
for i in range(n):
    for j in range(n):
        if i != j:
            print(i, j, torch.cuda.can_device_access_peer(i, j))
print(torch.cuda.get_device_properties(0))
PY

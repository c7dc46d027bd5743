#!/bin/bash
# The current GPU job (overwritten per gpurun call; outputs land in gpurun_out/, the ones worth
# keeping are copied to profiles/).  r5v (4 GPUs): the driver's 1-GPU suite + smoke on the
# new default (L128 band), bench lines N=1/2/4 + GoogLeNet, the N=1 launch list, ncu of the
# 128-byte-line two-shot (stepped N=4 on one GPU; N=2 across GPUs with NVLink counters).
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -x -q > $O/r5v_pytest_gpu_1gpu.log 2>&1; echo "suite rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r5v_smoke.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/r5v_bench1.json 2> $O/r5v_bench1.err; echo "b1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > $O/r5v_bench1_ref.json 2> $O/r5v_bench1_ref.err; echo "b1ref rc=$?"
T2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
T4="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29841 bench.py --gpus 2 --no-cpu-baseline > $O/r5v_bench2.json 2> $O/r5v_bench2.err; echo "b2 rc=$?"
timeout 900 $T4 --master-port 29842 bench.py --gpus 4 --no-cpu-baseline > $O/r5v_bench4.json 2> $O/r5v_bench4.err; echo "b4 rc=$?"
timeout 900 $T4 --master-port 29843 bench.py --gpus 4 --no-cpu-baseline --workload googlenet > $O/r5v_gbench4.json 2> $O/r5v_gbench4.err; echo "g4 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/r5v_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/r5v_ncu_launches.log 2>&1; echo "launches rc=$?"
# ncu of TWOSHOT_L128: fc8-size (16 MB) and conv3-size layers, stepped
for el in 4097000 885120; do
  cmd="python tools/ncu_stepped.py --world 4 --elems $el --variants twoshot_l128 --iters 2 --check"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd > $O/r5v_plain_l128_$el.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"k_twoshot_l128" -s 12 -c 6 -o $O/r5v_ncu_l128_$el $cmd > $O/r5v_ncu_l128_$el.log 2>&1
  echo "ncu l128 $el rc=$?"
  ncu -i $O/r5v_ncu_l128_$el.ncu-rep --page raw --csv > $O/r5v_ncu_l128_${el}_raw.csv 2>/dev/null
  ncu -i $O/r5v_ncu_l128_$el.ncu-rep --page details --csv > $O/r5v_ncu_l128_${el}_details.csv 2>/dev/null
  rm -f $O/r5v_ncu_l128_$el.ncu-rep
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
cmd="python tools/ncu_stepped.py --world 2 --devices 0,1 --elems 4097000 --variants twoshot_l128 --iters 2 --check"
timeout 300 $cmd > $O/r5v_plain_nvl_l128.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none --devices 0 --kernel-name-base demangled -k regex:"k_twoshot_l128" \
    --csv $cmd > $O/r5v_ncu_nvl_l128.csv 2> $O/r5v_ncu_nvl_l128.err; echo "nvl l128 rc=$?"
echo done

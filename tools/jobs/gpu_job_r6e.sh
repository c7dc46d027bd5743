#!/bin/bash
# r6e (4 GPUs): warp-specialised owner_tma (producer thread + consumer warps, full/done
# mbarriers per stage): parity (1 GPU stepped, 4 GPUs concurrent), ncu of the stepped bulk
# and cet owner kernels (vs r6a 253 us / r6c 26 us), sweeps, in-step N=4 ce vs bulk vs cet.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6e
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -m gpu -x -q -k "bulk or cet or ceb or benched" > $O/${R}_pytest_1gpu.log 2>&1; echo "suite1 rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -x -q -k "bulk or cet or ceb" > $O/${R}_pytest_4gpus.log 2>&1; echo "suite4 rc=$?"
FC6=37752832
run() {  # name variants regex skip count [ctas]
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5 ctas=${6:-0}
  local cmd="python tools/ncu_stepped.py --world 4 --elems $FC6 --variants $var --iters 2 --ctas $ctas"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd --check > $O/${R}_plain_$name.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $sk -c $cnt -o $O/${R}_ncu_$name $cmd > $O/${R}_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i $O/${R}_ncu_$name.ncu-rep --page raw --csv > $O/${R}_ncu_${name}_raw.csv 2>/dev/null
  ncu -i $O/${R}_ncu_$name.ncu-rep --page details --csv > $O/${R}_ncu_${name}_details.csv 2>/dev/null
  rm -f $O/${R}_ncu_$name.ncu-rep
}
run bulk4 twoshot_bulk "k_twoshot_bulk<.int.4," 8 5
run bulk4c48 twoshot_bulk "k_twoshot_bulk<.int.4," 8 5 48
run cet4 twoshot_cet "k_owner_tma<.int.4," 16 4
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/sweep.py --min-kb 4096 --max-mb 256 \
  --ctas 48 --variants twoshot_bulk > $O/${R}_sweep_n4_bulk48.jsonl 2> $O/${R}_sweep_n4_bulk48.err; echo "sweep rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
p=29900
b() { local name=$1; shift; p=$((p+1)); timeout 900 $TR --master-port $p $B "$@" > $O/${R}_bench4_$name.json 2> $O/${R}_bench4_$name.err; echo "$name rc=$?"; }
b ce_a
b bulk48_a --large bulk --large-ctas 48
b bulk32_a --large bulk --large-ctas 32
b cet64_a --large cet --large-ctas 64
b ce_b
b bulk48_b --large bulk --large-ctas 48
b bulk64_a --large bulk --large-ctas 64
b cet32_a --large cet --large-ctas 32
b ce_c
echo done

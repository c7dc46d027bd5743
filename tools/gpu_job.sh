#!/bin/bash
# r5z (4 GPUs): straight-line loads for whole vectors in the owner loops (+ slab_grad)
# (slab_grad): the 1-GPU suite, ncu of the stepped bulk / two-shot kernels (compare r5t),
# N=1 bench, N=4 sweep of the large layers and in-step AlexNet (ce default vs bulk 48).
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -x -q > $O/r5z_pytest_gpu_1gpu.log 2>&1; echo "suite rc=$?"
FC6=37752832
run() {  # name variants regex skip count
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5
  local cmd="python tools/ncu_stepped.py --world 4 --elems $FC6 --variants $var --iters 2"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd > $O/r5z_plain_$name.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $sk -c $cnt -o $O/r5z_ncu_$name $cmd > $O/r5z_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i $O/r5z_ncu_$name.ncu-rep --page raw --csv > $O/r5z_ncu_${name}_raw.csv 2>/dev/null
  ncu -i $O/r5z_ncu_$name.ncu-rep --page details --csv > $O/r5z_ncu_${name}_details.csv 2>/dev/null
  rm -f $O/r5z_ncu_$name.ncu-rep
}
run twoshot4 twoshot "k_twoshot<.int.4," 8 5
run bulk4 twoshot_bulk "k_twoshot_bulk<.int.4," 8 5
run ce4 twoshot_ce "k_owner_local<.int.4," 16 4
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/r5z_bench1.json 2> $O/r5z_bench1.err; echo "b1 rc=$?"
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 tools/sweep.py --min-kb 16384 --max-mb 256 \
  --variants twoshot,twoshot_ce > $O/r5z_sweep_n4.jsonl 2> $O/r5z_sweep_n4.err; echo "sweep rc=$?"
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29762 tools/sweep.py --min-kb 16384 --max-mb 256 \
  --ctas 48 --variants twoshot_bulk > $O/r5z_sweep_n4_bulk48.jsonl 2> $O/r5z_sweep_n4_bulk48.err; echo "sweep48 rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29863 $B > $O/r5z_bench4.json 2> $O/r5z_bench4.err; echo "b4 rc=$?"
timeout 900 $TR --master-port 29864 $B --large bulk --large-ctas 48 > $O/r5z_bench4_bulk48.json 2> $O/r5z_bench4_bulk48.err; echo "b4bulk rc=$?"
echo done

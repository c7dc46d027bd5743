#!/bin/bash
# r6b (4 GPUs; r6a had a port typo): TMA-fed owner fold in TWOSHOT_BULK (owner_tma): bulk parity (1 and 4 GPUs),
# ncu of the stepped bulk kernel (owner phase vs r5z's 395 us), N=4 sweeps at 24/48 CTAs,
# in-step AlexNet N=4: ce default vs bulk 24 / 48 (/ lean 48).
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -x -q -k "bulk" > $O/${R}_pytest_bulk_4gpus.log 2>&1; echo "suite4 rc=$?"
FC6=37752832
run() {  # name variants regex skip count
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5
  local cmd="python tools/ncu_stepped.py --world 4 --elems $FC6 --variants $var --iters 2"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd > $O/${R}_plain_$name.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $sk -c $cnt -o $O/${R}_ncu_$name $cmd > $O/${R}_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i $O/${R}_ncu_$name.ncu-rep --page raw --csv > $O/${R}_ncu_${name}_raw.csv 2>/dev/null
  ncu -i $O/${R}_ncu_$name.ncu-rep --page details --csv > $O/${R}_ncu_${name}_details.csv 2>/dev/null
  rm -f $O/${R}_ncu_$name.ncu-rep
}
for c in 24 48; do
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700+c)) tools/sweep.py --min-kb 4096 --max-mb 256 \
  --ctas $c --variants twoshot_bulk > $O/${R}_sweep_n4_bulk$c.jsonl 2> $O/${R}_sweep_n4_bulk$c.err; echo "sweep$c rc=$?"
done
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29863 $B > $O/${R}_bench4.json 2> $O/${R}_bench4.err; echo "b4 rc=$?"
for c in 24 48; do
timeout 900 $TR --master-port $((29800+c)) $B --large bulk --large-ctas $c > $O/${R}_bench4_bulk$c.json 2> $O/${R}_bench4_bulk$c.err; echo "b4bulk$c rc=$?"
done
timeout 900 $TR --master-port 29880 $B --large bulk --large-ctas 48 --xflags bulk_lean > $O/${R}_bench4_bulk48lean.json 2> $O/${R}_bench4_bulk48lean.err; echo "b4lean rc=$?"
timeout 900 $TR --master-port 29864 $B > $O/${R}_bench4_again.json 2> $O/${R}_bench4_again.err; echo "b4again rc=$?"
B2="bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29865 $B2 > $O/${R}_bench2.json 2> $O/${R}_bench2.err; echo "b2 rc=$?"
timeout 900 $TR2 --master-port 29866 $B2 --large bulk --large-ctas 24 > $O/${R}_bench2_bulk24.json 2> $O/${R}_bench2_bulk24.err; echo "b2bulk24 rc=$?"
echo done

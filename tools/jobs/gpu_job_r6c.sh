#!/bin/bash
# r6c (4 GPUs): TWOSHOT_CE with the TMA-fed owner fold on a capped grid (twoshot_cet /
# --large cet): parity (1 GPU stepped + 4 GPUs concurrent + graphs), ncu of the stepped
# k_owner_tma vs k_owner_local, N=4 sweep, in-step AlexNet N=4 and N=2: ce vs cet caps.
cd "$(dirname "$0")/../.." || exit 1
O=gpurun_out
R=r6c
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -m gpu -x -q -k "cet or benched" > $O/${R}_pytest_1gpu.log 2>&1; echo "suite1 rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "cet" > $O/${R}_pytest_4gpus.log 2>&1; echo "suite4 rc=$?"
FC6=37752832
run() {  # name variants regex skip count
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5
  local cmd="python tools/ncu_stepped.py --world 4 --elems $FC6 --variants $var --iters 2"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd --check > $O/${R}_plain_$name.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $sk -c $cnt -o $O/${R}_ncu_$name $cmd > $O/${R}_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i $O/${R}_ncu_$name.ncu-rep --page raw --csv > $O/${R}_ncu_${name}_raw.csv 2>/dev/null
  ncu -i $O/${R}_ncu_$name.ncu-rep --page details --csv > $O/${R}_ncu_${name}_details.csv 2>/dev/null
  rm -f $O/${R}_ncu_$name.ncu-rep
}
run cet4 twoshot_cet "k_owner_tma<.int.4," 16 4
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/sweep.py --min-kb 4096 --max-mb 256 \
  --variants twoshot_ce,twoshot_cet > $O/${R}_sweep_n4.jsonl 2> $O/${R}_sweep_n4.err; echo "sweep rc=$?"
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29863 $B > $O/${R}_bench4.json 2> $O/${R}_bench4.err; echo "b4 rc=$?"
for c in 16 32 64; do
timeout 900 $TR --master-port $((29800+c)) $B --large cet --large-ctas $c > $O/${R}_bench4_cet$c.json 2> $O/${R}_bench4_cet$c.err; echo "b4cet$c rc=$?"
done
timeout 900 $TR --master-port 29864 $B > $O/${R}_bench4_again.json 2> $O/${R}_bench4_again.err; echo "b4again rc=$?"
B2="bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline"
TR2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29865 $B2 > $O/${R}_bench2.json 2> $O/${R}_bench2.err; echo "b2 rc=$?"
timeout 900 $TR2 --master-port 29866 $B2 --large cet > $O/${R}_bench2_cet.json 2> $O/${R}_bench2_cet.err; echo "b2cet rc=$?"
echo done

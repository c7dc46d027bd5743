#!/bin/bash
# The current GPU job (overwritten per gpurun call; outputs land in gpurun_out/, the ones worth
# keeping are copied to profiles/).  r5u (4 GPUs): TWOSHOT_L128 at 64-256 MB; in-step AlexNet /
# GoogLeNet with the 128-byte-line two-shot for mid-size (and all) layers; configs[0]/[1] lines.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n \
    tools/sweep.py --min-kb 65536 --max-mb 256 --variants twoshot_l128,twoshot,twoshot_ce,nccl > $O/r5u_sweep_large_n$n.jsonl 2> $O/r5u_sweep_large_n$n.err
  echo "sweep n=$n rc=$?"
done
TR="torchrun --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline"
timeout 900 $TR --master-port 29821 $B --l128 65537:1048576 > $O/r5u_bench4_l128mid.json 2> $O/r5u_bench4_l128mid.err; echo "b1 rc=$?"
timeout 900 $TR --master-port 29822 $B --l128 65537:4000000000 > $O/r5u_bench4_l128all.json 2> $O/r5u_bench4_l128all.err; echo "b2 rc=$?"
timeout 900 $TR --master-port 29823 $B > $O/r5u_bench4_ce.json 2> $O/r5u_bench4_ce.err; echo "b3 rc=$?"
timeout 900 $TR --master-port 29824 $B --workload googlenet > $O/r5u_gbench4.json 2> $O/r5u_gbench4.err; echo "g1 rc=$?"
timeout 900 $TR --master-port 29825 $B --workload googlenet --l128 65537:1048576 > $O/r5u_gbench4_l128mid.json 2> $O/r5u_gbench4_l128mid.err; echo "g2 rc=$?"
T2="torchrun --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29826 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --l128 65537:1048576 > $O/r5u_bench2_l128mid.json 2> $O/r5u_bench2_l128mid.err; echo "b4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29827 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline > $O/r5u_bench2_ce.json 2> $O/r5u_bench2_ce.err; echo "b5 rc=$?"
# configs[0] LeNet-5 at 2 ranks, configs[1] cifar10_quick at 4 ranks: product arm + reference arm
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29828 bench.py --gpus 2 --workload lenet --steps 50 --warmup 10 > $O/r5u_lenet2.json 2> $O/r5u_lenet2.err; echo "l1 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29829 bench.py --gpus 2 --workload lenet --impl reference --steps 20 --warmup 3 > $O/r5u_lenet2_ref.json 2> $O/r5u_lenet2_ref.err; echo "l2 rc=$?"
timeout 900 $TR --master-port 29830 bench.py --gpus 4 --workload cifar10_quick --steps 50 --warmup 10 > $O/r5u_cifar4.json 2> $O/r5u_cifar4.err; echo "c1 rc=$?"
timeout 900 $TR --master-port 29831 bench.py --gpus 4 --workload cifar10_quick --impl reference --steps 20 --warmup 3 > $O/r5u_cifar4_ref.json 2> $O/r5u_cifar4_ref.err; echo "c2 rc=$?"
echo done

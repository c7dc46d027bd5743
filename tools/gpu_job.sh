#!/bin/bash
# The current GPU job (overwritten per gpurun call; the outputs land in gpurun_out/ and the
# ones worth keeping are copied to profiles/).  r5t (2 GPUs): ncu of the exchange kernels
# stepped on one GPU (N=4 emulated, --set full) and across two GPUs (N=2, NVLink byte
# counters), compute-sanitizer on the stepped exchanges, the 2-GPU multi/stress suite.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
FC6=37752832

# 1. ncu --set full, N=4 emulated on GPU 0 (each command first exits 0 without ncu)
run() {  # name variants regex skip count [elems]
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5 el=${6:-$FC6}
  local cmd="python tools/ncu_stepped.py --world 4 --elems $el --variants $var --iters 2"
  CUDA_VISIBLE_DEVICES=0 timeout 300 $cmd > $O/r5t_plain_$name.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$rx" -s $sk -c $cnt -o $O/r5t_ncu_$name $cmd > $O/r5t_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  # the .ncu-rep files are tens of MB: keep the text pages, drop the report (64 MiB pull cap)
  ncu -i $O/r5t_ncu_$name.ncu-rep --page details --csv > $O/r5t_ncu_${name}_details.csv 2>/dev/null
  ncu -i $O/r5t_ncu_$name.ncu-rep --page raw --csv > $O/r5t_ncu_${name}_raw.csv 2>/dev/null
  rm -f $O/r5t_ncu_$name.ncu-rep
}
run twoshot4 twoshot "k_twoshot<.int.4," 8 5
run bulk4 twoshot_bulk "k_twoshot_bulk<.int.4," 8 5
run ce4 twoshot_ce "k_owner_local<.int.4," 16 4
run ll4 oneshot_ll "k_oneshot_ll<.int.4>" 8 5 65536
run oneshot4 oneshot "k_oneshot<.int.4," 8 5 262144
run tree4 tree "k_tree_(up|down)<" 8 6

# 2. NVLink bytes: N=2 stepped across GPUs 0 and 1 (push / owner phases never wait on a
#    peer when launched in this order); ncu profiles device 0's launches only
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for v in twoshot twoshot_bulk oneshot tree; do
  el=$FC6; [ $v = oneshot ] && el=262144
  cmd="python tools/ncu_stepped.py --world 2 --devices 0,1 --elems $el --variants $v --iters 2 --check"
  timeout 300 $cmd > $O/r5t_plain_nvl_$v.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --devices 0 --kernel-name-base demangled -k regex:"k_(twoshot|oneshot|tree)" \
      --csv $cmd > $O/r5t_ncu_nvl_$v.csv 2> $O/r5t_ncu_nvl_$v.err
  echo "nvl $v rc=$?"
done

# 3. compute-sanitizer on the stepped exchanges (small layers, every variant, checked vs oracle)
SM="520,25050,400500,5010"
for tool in memcheck racecheck synccheck; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 compute-sanitizer --tool $tool --kernel-name kns=pgx --print-limit 50 \
      python tools/ncu_stepped.py --world 4 --elems $SM --variants twoshot,oneshot,oneshot_ll,twoshot_bulk,twoshot_ce,tree \
      --iters 2 --check > $O/r5t_sanitizer_$tool.full 2>&1
  echo "sanitizer $tool rc=$?"
  head -c 200000 $O/r5t_sanitizer_$tool.full > $O/r5t_sanitizer_$tool.log; rm -f $O/r5t_sanitizer_$tool.full
done

# 4. the 2-GPU multi / stress suite with test ids in the log
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -rA -q > $O/r5t_pytest_multi_4gpus.log 2>&1
echo "pytest rc=$?"
echo done

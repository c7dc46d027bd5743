#!/bin/bash
# 1-GPU job: the driver's GPU suite, then ncu captures of the exchange kernels stepped on one
# GPU (N=4 emulated; each command first exits 0 without ncu).  r5q.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
# (suite ran in r5q)



FC6=37752832
run() {  # name variants regex skip count [elems]
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5 el=${6:-$FC6}
  local cmd="python tools/ncu_stepped.py --world 4 --elems $el --variants $var --iters 2"
  timeout 300 $cmd > $O/r5q_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" -s $sk -c $cnt \
      -o $O/r5q_ncu_$name $cmd > $O/r5q_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
}
run twoshot4 twoshot "k_twoshot<.int.4," 8 5
run bulk4 twoshot_bulk "k_twoshot_bulk<.int.4," 8 5
run ce4 twoshot_ce "k_owner_local<.int.4," 16 4
run ll4 oneshot_ll "k_oneshot_ll<.int.4>" 8 5 65536
run oneshot4 oneshot "k_oneshot<.int.4," 8 5 262144

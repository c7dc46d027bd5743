#!/bin/bash
# 1-GPU job: the driver's GPU suite, then ncu captures of the exchange kernels stepped on one
# GPU (N=4 emulated; each command first exits 0 without ncu).  r5o.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r5o_pytest_gpu_1gpu.log 2>&1
echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r5o_smoke.log 2>&1
echo "smoke rc=$?"
FC6=37752832
run() {  # name variants regex skip count [elems]
  local name=$1 var=$2 rx=$3 sk=$4 cnt=$5 el=${6:-$FC6}
  local cmd="python tools/ncu_stepped.py --world 4 --elems $el --variants $var --iters 2"
  timeout 300 $cmd > $O/r5o_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" -s $sk -c $cnt \
      -o $O/r5o_ncu_$name $cmd > $O/r5o_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
}
run twoshot4 twoshot "k_twoshot<4" 8 5
run bulk4 twoshot_bulk "k_twoshot_bulk<4" 8 5
run ce4 twoshot_ce "k_owner_local<4" 16 4
run ll4 oneshot_ll "k_oneshot_ll<4" 8 5 65536
run oneshot4 oneshot "k_oneshot<4" 8 5 262144

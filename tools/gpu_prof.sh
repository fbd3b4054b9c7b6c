#!/bin/bash
# Isolated phase times (XRL_SERIAL=1 bench) + ncu --set full of selected kernels.
# usage: KERNELS="k_m2l_tc|k_p2p" LEAF=352 tools/gpu_prof.sh <tag>
T=${1:-prof}
O=gpurun_out/$T
mkdir -p $O
L=${LEAF:-352}
K=${KERNELS:-k_m2l_tc|k_p2p}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
XRL_SERIAL=1 timeout 600 python bench.py --steps 10 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 > $O/bench_serial.log 2>&1; echo "bench serial rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-2} -o $O/prof_full python tools/prof_mvm.py 4 4 $L > $O/ncu.log 2>&1; echo "ncu full rc=$?" >> $O/status.txt
cat $O/status.txt

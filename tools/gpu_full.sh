#!/bin/bash
# One GPU pass: build, smoke, gpu tests, default bench, launch list of the bench command, ncu --set full of the hot kernels.
# usage: tools/gpu_full.sh [tag]   (results under gpurun_out/<tag>/)
T=${1:-run}
O=gpurun_out/$T
mkdir -p $O
L=${LEAF:-384}
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1; nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
if [ "${TESTS:-1}" = "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q -s --durations=40 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
timeout 1200 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
if [ "${NCU:-1}" = "1" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/status.txt
# k_m2l_tc also runs the M2M and L2L passes (3 launches per MVM): skip 4 to capture the second MVM's M2L; fusion off (pure M2L)
for KS in k_m2l_tc:4 k_p2p:1 k_near_rg:1 k_l2p_leaf:1 k_m2p:1 k_p2m:1; do
K=${KS%%:*}; SK=${KS##*:}
XRL_FUSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$|::${K}\$|${K}\(|${K}<" -s $SK -c 1 -o $O/full_$K python tools/prof_mvm.py 4 3 $L > $O/ncu_$K.log 2>&1; echo "ncu full $K rc=$?" >> $O/status.txt
done
fi
cat $O/status.txt

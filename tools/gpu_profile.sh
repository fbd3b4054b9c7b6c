#!/bin/bash
# Round profiles for the bench configuration: launch list of bench.py + full ncu of the hot kernels.
mkdir -p gpurun_out
L=${LEAF:-512}
timeout 900 python bench.py --steps 3 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 > gpurun_out/bench_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/prof_mvm.py 4 2 $L > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_m2l|k_p2p|k_near_spmv|k_l2p_m2p|k_p2m|k_m2m|k_l2l" -s 20 -c 14 -o gpurun_out/prof_full python tools/prof_mvm.py 4 2 $L > gpurun_out/ncu.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

#!/bin/bash
mkdir -p gpurun_out
for L in 64 128 256 512; do
  timeout 600 python bench.py --steps 5 --warmup 3 --leaf $L --no-cpu-baseline > gpurun_out/bench_leaf$L.log 2>&1; echo "bench leaf$L rc=$?" >> gpurun_out/status.txt
done
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/prof_mvm.py 4 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l|k_p2p|k_near_spmv" -s 3 -c 3 -o gpurun_out/prof_r1d python tools/prof_mvm.py 4 2 > gpurun_out/ncu.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

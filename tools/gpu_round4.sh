#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for L in 64 128 256 512; do
timeout 600 python bench.py --steps 5 --warmup 3 --leaf $L --no-cpu-baseline > gpurun_out/bench_tc_leaf$L.log 2>&1; echo "bench tc leaf$L rc=$?" >> gpurun_out/status.txt
done
XRL_M2L_SIMT=1 timeout 600 python bench.py --steps 5 --warmup 3 --leaf 128 --no-cpu-baseline > gpurun_out/bench_simt_leaf128.log 2>&1; echo "bench simt rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/prof_mvm.py 4 2 128 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_tc" -s 1 -c 1 -o gpurun_out/prof_tc python tools/prof_mvm.py 4 2 128 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

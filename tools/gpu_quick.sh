#!/bin/bash
# quick: parity tests + bench at given leaves (LEAVES env)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for L in ${LEAVES:-256 512}; do
timeout 600 python bench.py --steps 5 --warmup 3 --leaf $L --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_leaf$L.log 2>&1; echo "bench leaf$L rc=$?" >> gpurun_out/status.txt
done
cat gpurun_out/status.txt

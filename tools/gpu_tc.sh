#!/bin/bash
mkdir -p gpurun_out
XRL_M2L_TC=1 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_tc.log 2>&1; echo "smoke tc rc=$?" >> gpurun_out/status.txt
if grep -q "rel L2" gpurun_out/smoke_tc.log; then
XRL_M2L_TC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full or sampled or ragged or clustered" > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc rc=$?" >> gpurun_out/status.txt
for L in 64 128 256 512; do
XRL_M2L_TC=1 timeout 300 python bench.py --steps 10 --warmup 3 --leaf $L --no-cpu-baseline --gmres-iters 0 > gpurun_out/bench_tc_leaf$L.log 2>&1; echo "bench tc leaf$L rc=$?" >> gpurun_out/status.txt
done
fi
cat gpurun_out/status.txt

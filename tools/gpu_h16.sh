#!/bin/bash
# FP16 M2L check: build, smoke, parity tests, short bench with and without the 3xFP16 M2L.
T=${1:-h16}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
XRL_M2L_TF32=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_tf32.log 2>&1; echo "bench tf32 rc=$?" >> $O/status.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
tail -n 3 $O/smoke.log $O/pytest_gpu.log
cat $O/status.txt

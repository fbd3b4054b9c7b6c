#!/bin/bash
# Iteration check: build, smoke, parity tests (fast subset unless TESTS=full), isolated phase times, short bench.
T=${1:-iter}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
if [ "${TESTS:-parity}" = "full" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
elif [ "${TESTS:-parity}" != "none" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
TAG=cur timeout 300 python tools/phase_times.py 4 ${LEAF:-384} 10 > $O/phases.json 2>> $O/err.log; echo "phases rc=$?" >> $O/status.txt
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 ${BENCH_ARGS} > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
tail -n 2 $O/smoke.log $O/pytest_gpu.log 2>/dev/null
cat $O/status.txt $O/phases.json

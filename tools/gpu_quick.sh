#!/bin/bash
# Quick GPU iteration: build, smoke canary, parity tests, short bench (+ optional extra command in $EXTRA).
# usage: tools/gpu_quick.sh <tag>
T=${1:-quick}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/status.txt
if [ $rc = 0 ]; then
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gmres-iters 0 ${BENCH_ARGS} > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
XRL_SCHED=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gmres-iters 0 ${BENCH_ARGS} > $O/bench_serial.log 2>&1; echo "bench serial rc=$?" >> $O/status.txt
XRL_SCHED=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gmres-iters 0 ${BENCH_ARGS} > $O/bench_sched1.log 2>&1; echo "bench sched1 rc=$?" >> $O/status.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
fi
tail -n 3 $O/smoke.log $O/pytest_gpu.log
cat $O/status.txt

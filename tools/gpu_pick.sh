#!/bin/bash
# P2P register-tile choice per task (XRL_P2P_PICK): parity tests, then isolated phase times and a short bench
# for each value.  usage: VALS="0 106" tools/gpu_pick.sh <tag>
T=${1:-pick}; O=gpurun_out/$T; rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout ${PT:-900} python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for v in ${VALS:-0 106}; do
XRL_P2P_PICK=$v XRL_FUSE=0 timeout 300 python tools/phase_times.py 4 384 20 > $O/phase_$v.log 2>&1; echo "phase $v rc=$?" >> $O/status.txt
XRL_P2P_PICK=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_$v.log 2>&1; echo "bench $v rc=$?" >> $O/status.txt
done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
tail -n 3 $O/pytest_gpu.log
cat $O/status.txt

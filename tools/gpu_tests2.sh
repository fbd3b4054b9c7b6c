#!/bin/bash
# GPU pass: build, smoke, the whole -m gpu suite (durations), a short default bench.
# usage: tools/gpu_tests2.sh <tag> [pytest -k expr]
T=${1:-t}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -s --durations=30 ${2:+-k "$2"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
fi
tail -n 5 $O/pytest_gpu.log
cat $O/status.txt

#!/bin/bash
# Sweep an env-selected kernel variant: VAR=<env name> VALS="0 1 2" tools/gpu_var.sh <tag>
T=${1:-var}; O=gpurun_out/$T; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for v in $VALS; do
env $VAR=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gmres-iters 0 ${BENCH_ARGS} > $O/bench_$v.log 2>&1; echo "bench $v rc=$?" >> $O/status.txt
done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
cat $O/status.txt

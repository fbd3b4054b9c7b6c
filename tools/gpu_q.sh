#!/bin/bash
# quick GPU iteration: build, selected tests (-k $K), short bench, optional ncu of one kernel ($NCUK)
T=${1:-q}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout ${PT:-900} python -m pytest ${TESTS:-tests} -m gpu -q -s -x ${K:+-k "$K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 ${BENCH_ARGS} > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
fi
if [ -n "$NCUK" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCUK -s ${NCUS:-2} -c 1 -o $O/full_$NCUK python tools/prof_mvm.py 4 3 352 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?" >> $O/status.txt; fi
tail -n 3 $O/pytest_gpu.log
cat $O/status.txt

#!/bin/bash
# leaf-size sweep of the default bench (short): tools/gpu_sweep.sh <tag> "256 384 512"
T=${1:-sweep}
O=gpurun_out/$T
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for L in ${2:-256 384 512 768}; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --leaf $L ${BENCH_ARGS} > $O/bench_leaf$L.log 2>&1; echo "leaf $L rc=$?" >> $O/status.txt
done
cat $O/status.txt

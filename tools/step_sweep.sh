#!/bin/bash
# Step-time variants: for each "flags|env" item, build with XRL_EXTRA_NVCC=flags and run a short bench with the
# given environment (e.g. "-DXRL_FUSE_WARPS=2|" or "|XRL_FUSE=0").   usage: tools/step_sweep.sh tag item ...
T=$1; shift
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
for IT in "$@"; do
  F="${IT%%|*}"; E="${IT#*|}"
  XRL_EXTRA_NVCC="$F" python -m paper_2409_12375_b200.build --force > $O/build.log 2>&1 || { echo "build failed: $F" >> $O/sweep.txt; continue; }
  env $E timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/b.log 2>>$O/err.log
  echo "== [$F] [$E] $(python tools/show_bench.py $O/b.log | cut -c1-200)" >> $O/sweep.txt
done
python -m paper_2409_12375_b200.build --force > $O/build.log 2>&1
cat $O/sweep.txt

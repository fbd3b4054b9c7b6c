#!/bin/bash
# Compile-time variants (XRL_EXTRA_NVCC flags): per variant the isolated phase times of config 4 (fusion off)
# and a short bench.   usage: tools/build_var.sh tag "flags1" "flags2" ...
T=$1; shift
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
i=0
for F in "$@"; do
  i=$((i+1))
  XRL_EXTRA_NVCC="$F" python -m paper_2409_12375_b200.build --force > $O/build_$i.log 2>&1 || { echo "build failed: $F" >> $O/sweep.txt; continue; }
  echo "== $F" >> $O/sweep.txt
  XRL_FUSE=0 timeout 300 python tools/phase_times.py 4 ${LEAF:-384} 20 >> $O/sweep.txt 2>>$O/err.log
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project ${PROJ:-0} > $O/bench_$i.log 2>&1
  python -c "
import json;b=json.loads([l for l in open('$O/bench_$i.log') if l.startswith('{')][0]);print('bench', b['ms_per_step'], b['timing']['ms_median'], b['value'], b.get('multi_gpu_projection',{}).get('speedup_vs_1gpu'))" >> $O/sweep.txt 2>>$O/err.log
done
python -m paper_2409_12375_b200.build --force > $O/build.log 2>&1
cat $O/sweep.txt

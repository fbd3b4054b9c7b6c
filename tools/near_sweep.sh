#!/bin/bash
# Near SpMV variants (compile-time flags): isolated phase times of config 4 for each, then an ncu capture of
# k_near_rg for the default build.   usage: tools/near_sweep.sh tag "flags1" "flags2" ...
T=$1; shift
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
for F in "$@"; do
  XRL_EXTRA_NVCC="$F" python -m paper_2409_12375_b200.build --force > $O/build.log 2>&1 || { echo "build failed: $F" >> $O/sweep.txt; continue; }
  echo "== $F $(TAG="$F" timeout 300 python tools/phase_times.py 4 ${LEAF:-384} 10 2>>$O/err.log)" >> $O/sweep.txt
done
python -m paper_2409_12375_b200.build --force > $O/build.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
XRL_FUSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near_rg" -s 1 -c 1 -o $O/full_k_near_rg python tools/prof_mvm.py 4 3 ${LEAF:-384} > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/sweep.txt
fi
cat $O/sweep.txt

#!/bin/bash
# ncu --set full of one kernel (first launch after SKIP) in tools/prof_mvm.py at config 4.
# usage: K=k_p2p SKIP=1 LEAF=352 tools/ncu_one.sh <tag>
T=${1:-one}; O=gpurun_out/$T; rm -rf $O; mkdir -p $O
L=${LEAF:-352}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$|::${K}\$|${K}\(" -s ${SKIP:-1} -c 1 -o $O/full_$K python tools/prof_mvm.py 4 3 $L > $O/ncu_$K.log 2>&1; echo "ncu full $K rc=$?" >> $O/status.txt
cat $O/status.txt

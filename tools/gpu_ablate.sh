#!/bin/bash
# M2L ablation timings (build with -DXRL_PROFILING_ABLATION; XRL_M2L_DBG 1 = no reductions, 2 = no A loads, 4 = no D reads)
T=${1:-abl}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
touch paper_2409_12375_b200/csrc/fmm.cu; XRL_EXTRA_NVCC="-DXRL_PROFILING_ABLATION" python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
for D in 0 1 2 3 4 5 7; do
  TAG=h16_dbg$D XRL_M2L_DBG=$D timeout 300 python tools/phase_times.py 4 384 10 >> $O/times.jsonl 2>> $O/err.log
  TAG=tf32_dbg$D XRL_M2L_TF32=1 XRL_M2L_DBG=$D timeout 300 python tools/phase_times.py 4 384 10 >> $O/times.jsonl 2>> $O/err.log
done
touch paper_2409_12375_b200/csrc/fmm.cu; python -c "import __graft_entry__ as g; g.build()" > $O/build2.log 2>&1
cat $O/times.jsonl

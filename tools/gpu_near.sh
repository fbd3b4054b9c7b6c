#!/bin/bash
# near SpMV iteration: parity tests touching the near path + short bench + ncu of k_near_blk
T=${1:-near}
O=gpurun_out/$T
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -s -x -k "near or full_mvm_config1 or special or schedules or single_leaf or tiny" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_near_blk -s 2 -c 1 -o $O/full_k_near_blk python tools/prof_mvm.py 4 3 352 > $O/ncu_near.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
fi
tail -n 3 $O/pytest_gpu.log
cat $O/status.txt

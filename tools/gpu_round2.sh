#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/prof_mvm.py 4 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_m2l|k_p2p|k_p2l|k_near_spmv|k_l2p_m2p" -s 5 -c 5 -o gpurun_out/prof_r1c python tools/prof_mvm.py 4 2 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

# fused near-in-P2P: smoke, parity (incl. full-size), bench fused vs separate
O=gpurun_out/${1:-q32}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_fused.log 2>&1; echo "bench fused rc=$?" >> $O/status.txt
XRL_NEAR_FUSE=0 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_sep.log 2>&1; echo "bench sep rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_mvm_4096" > $O/fullsize.log 2>&1; echo "fullsize rc=$?" >> $O/status.txt
cat $O/status.txt

# tensor-core P2P bring-up: smoke, parity, bench (TC vs SIMT P2P)
O=gpurun_out/${1:-q29}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_tc.log 2>&1; echo "bench tc rc=$?" >> $O/status.txt
XRL_P2P_TC=0 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_simt.log 2>&1; echo "bench simt rc=$?" >> $O/status.txt
cat $O/status.txt

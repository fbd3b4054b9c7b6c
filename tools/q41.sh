# root cube at the bounding-box corner: halo diag, parity subset, bench (with the 8-rank projection)
O=gpurun_out/${1:-q41}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/halo_diag.py 4 2 384 > $O/halo2.log 2>&1
timeout 300 python tools/halo_diag.py 4 8 384 > $O/halo8.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 1200 python tools/vrank_projection.py --config 4 --ks 1,2,4,8 --out $O/cfg4.json > $O/cfg4.log 2>&1; echo "proj rc=$?" >> $O/status.txt
cat $O/status.txt

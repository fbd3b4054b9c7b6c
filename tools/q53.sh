# GMRES single-sync step (all parts): solver tests, GMRES projection, bench GMRES probe
O=gpurun_out/${1:-q53}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > $O/solver.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 1500 python tools/gmres_projection.py --out $O/gmres.json > $O/gmres.log 2>&1; echo "gmres rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-leaf64 --project 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
cat $O/status.txt

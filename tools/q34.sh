# paired triples: parity tests + timing
O=gpurun_out/${1:-q34}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "paired or schedules or host" > $O/pair_tests.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 600 python tools/pair_timing.py --out $O/pair.json > $O/pair.log 2>&1; echo "timing rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
cat $O/status.txt

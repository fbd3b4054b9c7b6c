# concurrent-add schedule: tests + bench default vs XRL_SCHED=3
O=gpurun_out/${1:-q39}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "schedules or paired or config1 or vranks or virtual" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_fork.log 2>&1; echo "bench fork rc=$?" >> $O/status.txt
XRL_SCHED=3 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_conc.log 2>&1; echo "bench conc rc=$?" >> $O/status.txt
XRL_SCHED=3 XRL_FUSE=0 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_conc_nofuse.log 2>&1; echo "bench conc nofuse rc=$?" >> $O/status.txt
cat $O/status.txt

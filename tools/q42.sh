# leaf sweep on config 4 with the corner-aligned root cube; configs 3 and 5 at the default leaf
O=gpurun_out/${1:-q42}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for L in 320 352 416 448 512; do
  timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 --leaf $L > $O/bench_leaf$L.log 2>&1; echo "leaf $L rc=$?" >> $O/status.txt
done
for C in 3 5; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_cfg$C.log 2>&1; echo "cfg $C rc=$?" >> $O/status.txt
done
cat $O/status.txt

O=gpurun_out/lf1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for L in 320 352 384 416 448; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 --leaf $L > $O/b$L.log 2>>$O/err.log
  echo "leaf $L $(python tools/show_bench.py $O/b$L.log | cut -c1-120)" >> $O/sweep.txt
done
cat $O/sweep.txt

# P2P tuning sweep: each variant rebuilt with XRL_EXTRA_NVCC, isolated P2P + step time
O=gpurun_out/${1:-q40}; mkdir -p $O
for V in "base:" "u1:-DXRL_P2P_UNROLL=1" "u4:-DXRL_P2P_UNROLL=4" "t6:-DXRL_P2P_TPT=6" "cut192:-DXRL_P2P_CUT=192" "cut320:-DXRL_P2P_CUT=320"; do
  N=${V%%:*}; F=${V#*:}
  XRL_EXTRA_NVCC="$F" python -c "from paper_2409_12375_b200 import build; build.build(force=True)" > $O/build_$N.log 2>&1
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 > $O/bench_$N.log 2>&1; echo "$N rc=$?" >> $O/status.txt
done
python -c "from paper_2409_12375_b200 import build; build.build(force=True)" > $O/build_final.log 2>&1
cat $O/status.txt

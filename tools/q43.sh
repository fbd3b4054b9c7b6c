# partition weight sweep (8 virtual ranks of config 4): per-rank max / mean and projection
O=gpurun_out/${1:-q43}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for V in "base:2.0,0.7,0.006" "m1:1.0,0.7,0.006" "m3:3.0,0.7,0.006" "p2:2.0,1.5,0.006" "n2:2.0,0.7,0.02" "m4:4.0,0.7,0.006"; do
  N=${V%%:*}; W=${V#*:}
  XRL_PART_W=$W timeout 900 python tools/vrank_projection.py --config 4 --ks 8 --reps 5 --out $O/p_$N.json > $O/p_$N.log 2>&1; echo "$N rc=$?" >> $O/status.txt
done
cat $O/status.txt

# schedule variants at 8 virtual ranks of config 4
O=gpurun_out/${1:-q44}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for V in "base:" "fuse8:XRL_FUSE_MAXWORLD=8" "late:XRL_SCHED=2" "late_fuse8:XRL_SCHED=2 XRL_FUSE_MAXWORLD=8"; do
  N=${V%%:*}; E=${V#*:}
  env $E timeout 900 python tools/vrank_projection.py --config 4 --ks 8 --reps 5 --out $O/p_$N.json > $O/p_$N.log 2>&1; echo "$N rc=$?" >> $O/status.txt
done
cat $O/status.txt

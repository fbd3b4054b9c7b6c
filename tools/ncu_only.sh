O=gpurun_out/s2c2; mkdir -p $O; L=512
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for KS in k_m2l_tc:5 k_l2p_leaf:1 k_m2p:1; do
K=${KS%%:*}; SK=${KS##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$|::${K}\$|${K}\(" -s $SK -c 1 -o $O/full_$K python tools/prof_mvm.py 4 3 $L > $O/ncu_$K.log 2>&1; echo "ncu full $K rc=$?" >> $O/status.txt
done
cat $O/status.txt

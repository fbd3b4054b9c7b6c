# ncu --set full of one k_p2p_tc launch (config 4, leaf 384)
O=gpurun_out/${1:-q30}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
XRL_FUSE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_p2p_tc" -c 1 -o $O/full_k_p2p_tc python tools/prof_mvm.py 4 2 384 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
cat $O/status.txt

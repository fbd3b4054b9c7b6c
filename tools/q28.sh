O=gpurun_out/q28; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
XRL_FUSE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_m2l_tc" -s 4 -c 1 -o $O/full_k_m2l_tc python tools/prof_mvm.py 4 3 384 > $O/ncu_k_m2l_tc.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
timeout 1500 python tools/gmres_projection.py --out $O/gmres.json > $O/gmres.log 2>&1; echo "gmres rc=$?" >> $O/status.txt
cat $O/status.txt

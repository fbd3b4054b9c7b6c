# final measurement batch: projections, GMRES projection, Table IV, pair timing
O=gpurun_out/${1:-q54}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/vrank_projection.py --config 4 --ks 1,2,4,8 --out $O/proj_cfg4.json > $O/cfg4.log 2>&1; echo "cfg4 rc=$?" >> $O/status.txt
timeout 900 python tools/vrank_projection.py --config 3 --ks 1,8 --out $O/proj_cfg3.json > $O/cfg3.log 2>&1; echo "cfg3 rc=$?" >> $O/status.txt
timeout 1800 python tools/vrank_projection.py --config 5 --ks 1,8 --reps 3 --out $O/proj_cfg5.json > $O/cfg5.log 2>&1; echo "cfg5 rc=$?" >> $O/status.txt
timeout 2000 python tools/gmres_projection.py --out $O/gmres_projection.json > $O/gmres.log 2>&1; echo "gmres rc=$?" >> $O/status.txt
timeout 2400 python tools/table4.py --configs 1,2,4 --out $O/table4.json > $O/table4.log 2>&1; echo "table4 rc=$?" >> $O/status.txt
timeout 600 python tools/pair_timing.py --out $O/pair_timing.json > $O/pair.log 2>&1; echo "pair rc=$?" >> $O/status.txt
cat $O/status.txt

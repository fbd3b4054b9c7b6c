# final measurement batch after the tree-placement change: projections (cfg 4 sweep, cfg 3/5 at 8), GMRES, pair timing
O=gpurun_out/${1:-q48}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/vrank_projection.py --config 4 --ks 1,2,4,8 --out $O/cfg4.json > $O/cfg4.log 2>&1; echo "cfg4 rc=$?" >> $O/status.txt
timeout 900 python tools/vrank_projection.py --config 3 --ks 1,8 --out $O/cfg3.json > $O/cfg3.log 2>&1; echo "cfg3 rc=$?" >> $O/status.txt
timeout 1800 python tools/vrank_projection.py --config 5 --ks 1,8 --reps 3 --out $O/cfg5.json > $O/cfg5.log 2>&1; echo "cfg5 rc=$?" >> $O/status.txt
timeout 1500 python tools/gmres_projection.py --out $O/gmres.json > $O/gmres.log 2>&1; echo "gmres rc=$?" >> $O/status.txt
timeout 600 python tools/pair_timing.py --out $O/pair.json > $O/pair.log 2>&1; echo "pair rc=$?" >> $O/status.txt
cat $O/status.txt

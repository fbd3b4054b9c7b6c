O=gpurun_out/${1:-q35}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/pair_timing.py --out $O/pair.json > $O/pair.log 2>&1; echo "timing rc=$?" >> $O/status.txt
cat $O/status.txt

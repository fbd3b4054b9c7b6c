# GMRES iteration projection (config 4) with the single-GPU solver beside it
O=gpurun_out/${1:-q31}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/gmres_projection.py --out $O/gmres.json > $O/gmres.log 2>&1; echo "gmres rc=$?" >> $O/status.txt
cat $O/status.txt

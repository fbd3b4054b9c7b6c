# ILU(0) preconditioner: Table IV rows for configs 1, 2, 4
O=gpurun_out/${1:-q33}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/table4.py --configs 1,2,4 --only-ilu --out $O/table4_ilu.json > $O/table4_ilu.log 2>&1; echo "table4 rc=$?" >> $O/status.txt
cat $O/status.txt

#!/bin/bash
# Root-placement cost weight (XRL_COST_V, P2P pairs per V-list translation) x leaf size: short benches.
O=gpurun_out/${1:-cw1}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for W in ${WS:-1000 1500 2180}; do for L in ${LS:-352 384 416}; do
  XRL_COST_V=$W timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --gmres-iters 0 --no-leaf64 --project 0 --leaf $L > $O/b.log 2>>$O/err.log
  echo "w $W leaf $L $(python tools/show_bench.py $O/b.log | cut -c1-110) $(python -c "import json;d=[json.loads(l) for l in open('$O/b.log') if l.startswith('{')][0];c=d['config'];print(c['p2p_pairs'],c['m2l_translations'])")" >> $O/sweep.txt
done; done
cat $O/sweep.txt

# root placement chosen by the cost model: bench (leaf 384 + leaf 64 line), parity subset, setup times
O=gpurun_out/${1:-q45}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/setup_times.py 4 384 > $O/setup.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --gmres-iters 0 --project 0 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for C in 1 2 3 5; do timeout 600 python -c "
import sys; sys.path.insert(0,'.')
from inputs import meshes; from paper_2409_12375_b200 import xrl
m=meshes.make_config($C); ctx=xrl.Context(0)
for L in (64, 384):
    t=xrl.Tree(ctx, m.verts, m.tris, leaf_max=L); i=t.info(); print($C, L, i['root_lo'], i['n_p2p'], i['n_v_pairs'])
" >> $O/align.log 2>&1; done
cat $O/status.txt

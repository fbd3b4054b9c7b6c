# cost model over root shifts on the thin axis (config 4, leaf 384 and 64)
O=gpurun_out/${1:-q46}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for F in 0 0.001 0.002 0.004 0.006 0.008 0.012 0.016 0.024; do
XRL_ROOT_ALIGN=corner XRL_ROOT_SHIFT=$F timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from inputs import meshes; from paper_2409_12375_b200 import xrl
m=meshes.make_config(4); ctx=xrl.Context(0)
for L in (64, 384):
    t=xrl.Tree(ctx, m.verts, m.tris, leaf_max=L); i=t.info(); print('$F', L, i['n_p2p'], i['n_v_pairs'], round((i['n_p2p']*0.5e-9+i['n_v_pairs']*1.09e-6)*1e3,3), 'ms model')
" >> $O/shift.log 2>&1; done
cat $O/shift.log

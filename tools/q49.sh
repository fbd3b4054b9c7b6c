# cost model over x/y placements (config 4, leaf 384 and 64; the thin-axis search still runs per placement)
O=gpurun_out/${1:-q49}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for V in "0,0,0" "0.0156,0.0078,0.0078" "0.0156,0.0039,0.0117" "0.0156,0.0117,0.0039" "0.0313,0.0156,0.0156" "0.0313,0.0078,0.0234" "0.0078,0.0039,0.0039" "0.0625,0.0313,0.0313"; do
XRL_ROOT_XY=$V timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from inputs import meshes; from paper_2409_12375_b200 import xrl
m=meshes.make_config(4); ctx=xrl.Context(0)
for L in (384, 64):
    t=xrl.Tree(ctx, m.verts, m.tris, leaf_max=L); i=t.info(); print('$V', L, i['n_p2p'], i['n_v_pairs'], round(i['n_p2p']*0.5e-6+i['n_v_pairs']*1.09e-3,3), 'ms model')
" >> $O/xy.log 2>&1; done
cat $O/xy.log

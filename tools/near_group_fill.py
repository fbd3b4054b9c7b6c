"""Near-field pattern statistics for the row-group SpMV format: nonzeros per union column (gathers saved) and
bytes per nonzero for groups of G = 1, 2, 4, 8 consecutive Morton-ordered rows.  The pattern is the near
criterion d < eta max(D_k, D_l) (eta = 1.5, D = longest edge: an estimate, not the oracle's or the library's
pattern) found with a k-d tree on the FP64 centroids (no GPU).
    python tools/near_group_fill.py <config>"""
import numpy as np, time, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import meshes
ETA = 1.5
from scipy.spatial import cKDTree
cfg=int(sys.argv[1])
t=time.time(); m=meshes.make_config(cfg); print('mesh',m.n,time.time()-t)
P=m.verts[m.tris]
c=P.mean(1)
D=np.max([np.linalg.norm(P[:,a]-P[:,b],axis=1) for a,b in ((0,1),(1,2),(2,0))],axis=0)
lo=c.min(0); s=(c.max(0)-lo).max()*1.0001
q=np.floor((c-lo)/s*(1<<21)).astype(np.uint64)
def spread(v):
    v=v&np.uint64(0x1fffff)
    v=(v|(v<<np.uint64(32)))&np.uint64(0x1f00000000ffff)
    v=(v|(v<<np.uint64(16)))&np.uint64(0x1f0000ff0000ff)
    v=(v|(v<<np.uint64(8)))&np.uint64(0x100f00f00f00f00f)
    v=(v|(v<<np.uint64(4)))&np.uint64(0x10c30c30c30c30c3)
    v=(v|(v<<np.uint64(2)))&np.uint64(0x1249249249249249)
    return v
key=spread(q[:,0])|(spread(q[:,1])<<np.uint64(1))|(spread(q[:,2])<<np.uint64(2))
perm=np.argsort(key,kind='stable'); c=c[perm]; D=D[perm]
tr=cKDTree(c)
R=ETA*D.max()
t=time.time(); pairs=tr.query_pairs(R,output_type='ndarray'); print('pairs',len(pairs),time.time()-t)
i,j=pairs[:,0],pairs[:,1]
d2=((c[i]-c[j])**2).sum(1); ok=d2<(ETA*np.maximum(D[i],D[j]))**2
i,j=i[ok],j[ok]
rows=np.concatenate([i,j,np.arange(len(c))]); cols=np.concatenate([j,i,np.arange(len(c))])
nnz=len(rows); print('nnz',nnz,'per row',nnz/len(c))
for G in (1,2,4,8):
    u=np.unique((rows//G).astype(np.int64)*(1<<32)+cols).size
    print(f'G={G} union cols {u} fill {nnz/(u*G):.3f} gathers reduction {nnz/u:.2f}  bytes/nnz {(4*G+2)*u/nnz:.2f}')

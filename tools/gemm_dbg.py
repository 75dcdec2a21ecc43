import numpy as np, sys
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_1810_02719_b200 as G
import specmesh_oracle as O
ctx=G.Context(0)
for n,c in [(100,8),(100,20),(300,40),(300,64),(500,100),(2048,200),(600,33)]:
    b=np.random.default_rng(c).standard_normal((n,c))
    try:
        q=G.orthonormalize(b, ctx=ctx)
        print(n,c,'orth err',np.abs(q.T@q-np.eye(c)).max(), 'vs oracle', np.abs(q-O.orthonormalize(b)).max())
    except Exception as e:
        print(n,c,'ERR',e)
for n,c in [(300,60),(300,50),(300,120),(600,250)]:
    b=np.random.default_rng(c).standard_normal((n,c))
    q=G.orthonormalize(b, ctx=ctx)
    print(n,c,'orth err',np.abs(q.T@q-np.eye(c)).max(), 'vs oracle', np.abs(q-O.orthonormalize(b)).max())

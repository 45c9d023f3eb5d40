"""K2 v2 plan: lower bound on shared-memory wavefronts per LDS at C3 (busiest bank
degree / steps, per warp of 32 entry-sorted columns; CPU model with the C oracle
CountSketch, lane-pair splits ignored)."""
import numpy as np, sys
sys.path.insert(0,'.')
from oracle import skp_oracle as o
from paper_2605_09755_b200.sketching import substream
n,l,s=16384,4000,8
cols,signs=o.countsketch_c(7,n,l,s)
# entries per output column: list of j
byc=[[] for _ in range(l)]
for j in range(n):
    for c in cols[j]: byc[c].append(j)
cnt=np.array([len(x) for x in byc])
W=672; tot=0; LB=0; Ls=0; Ks=[]
for p in range(0,l,W):
    cs=np.arange(p,min(p+W,l)); cs=cs[np.argsort(-cnt[cs],kind='stable')]
    for w in range(0,len(cs),32):
        g=cs[w:w+32]; L=cnt[g].max()
        d=np.zeros(32,int)
        for c in g:
            for j in byc[c]: d[j&31]+=1
        Ks.append(max(0,d.max()-L)); Ls+=L; LB+=max(L,d.max())
print("warps",len(Ks),"mean L",Ls/len(Ks),"mean K",np.mean(Ks),"ideal wavefronts/LDS",LB/Ls)

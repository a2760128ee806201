import sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
cfg=get_config("C4"); xyz,tri=mesh_for(cfg)
h=DH2(xyz,tri,cfg["kappa"],cfg["m"],cfg["leaf"],cfg["eta1"],cfg["eta2"],device=-1)
h.set_option("lean_chunks",32)
bptr=h.export("lean_blk_ptr",np.int32); blk=h.export("lean_blk",np.int32)
Rr=h.export("bp_R_rows",np.int32)
blocks=h.export("blocks",np.int64).reshape(-1,3)
bp=h.export("basis_pairs",np.int64).reshape(-1,3)
bp_id={(int(t),int(c)):i for i,(_,t,c) in enumerate(bp)}
bpcs=h.export("blk_bpcs",np.int32)
k=125
b0=blk[bptr[0]:bptr[1]]
fl=0.0
for b in b0:
    t,s,c=blocks[b]; rt=Rr[bp_id[(int(t),int(c))]]; rs=Rr[bpcs[b]]
    fl+=8.0*(rt*k*k+rt*rs*k)
print("chunk0 blocks",len(b0),"model GF %.1f"%(fl/1e9))
dur=25.091712e-3
print("model TF/s %.2f"%(fl/dur/1e12), "frac of 37.07: %.3f"%(fl/dur/1e12/37.07))
act=19437623.351351; cyc=49062946.682432
# executed DMMA flops if 100% active == measured DMMA peak
print("counter-implied TF/s %.2f"%(act/cyc*37.07))

import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for, seeded_vector
from conftest import oracle_run
from oracle import ops
name=sys.argv[1]; ws=int(sys.argv[2])
cfg=get_config(name); xyz,tri=mesh_for(cfg)
h=DH2(xyz,tri,cfg['kappa'],cfg['m'],cfg['leaf'],cfg['eta1'],cfg['eta2'])
h.set_option('truncate_workspace', ws)
h.recompress(cfg['eps'])
rc=oracle_run(name)
x=seeded_vector(rc.st.n,1); yo=ops.matvec(rc,x,'orig')
print(name, 'ws',ws,'orig err %.2e'%(np.linalg.norm(h.matvec(x,0)-yo)/np.linalg.norm(yo)), 'recomp err %.2e'%(np.linalg.norm(h.matvec(x,1)-ops.matvec(rc,x,'recomp'))/np.linalg.norm(yo)))
rk=h.export('rank_row',np.int32); print('ranks gpu', rk[:10], 'orc', [rc.row.rank[k] for k in list(rc.row.rank)[:10]])
for nm, dt in (("normG2", np.float64), ("omega", np.float64), ("VR", np.complex128), ("Z_row", np.complex128), ("sigma_row", np.float64), ("C_row", np.complex128)):
    a = h.export(nm, dt)
    print(nm, "nonfinite", int(np.sum(~np.isfinite(a))), "of", a.size, "min|.| %.3e" % (np.min(np.abs(a)) if a.size else 0))

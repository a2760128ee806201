"""Distribution of sigma_i/sigma_1 per level on the GPU result (how many singular values per
pair lie above 1e-10, 1e-12, 1e-14 relative)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
h.recompress(cfg["eps"])
sig = h.export("sigma_row", np.float64); off = h.export("sig_off_row", np.int64); ns = h.export("nsig_row", np.int32)
lp = h.export("lev_ptr_row", np.int32)
for l in range(len(lp) - 1):
    a, b = lp[l], lp[l + 1]
    if b <= a:
        continue
    cnt = {t: [] for t in (1e-8, 1e-10, 1e-12, 1e-13, 1e-14)}
    for p in range(a, b):
        s = sig[off[p]:off[p] + ns[p]]
        if len(s) == 0:
            continue
        for t in cnt:
            cnt[t].append(int(np.sum(s > t * s[0])))
    print("level", l, "pairs", b - a, "nsig mean %.1f" % ns[a:b].mean(),
          " ".join("%g:%.1f" % (t, np.mean(v)) for t, v in cnt.items()))

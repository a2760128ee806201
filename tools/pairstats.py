"""Per-level statistics of a recompression on the GPU (ranks, singular-value counts, Jacobi sweeps)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
h.recompress(cfg["eps"])
for side in ("row", "col"):
    sw = h.export("sweeps_" + side, np.int32); lp = h.export("lev_ptr_" + side, np.int32)
    rk = h.export("rank_" + side, np.int32); zr = h.export("Z_rows_" + side, np.int32); ns = h.export("nsig_" + side, np.int32)
    for l in range(len(lp) - 1):
        a, b = lp[l], lp[l + 1]
        if b > a:
            print(side, l, b - a, "sweeps %.2f/%d" % (sw[a:b].mean(), sw[a:b].max()), "rank %.2f/%d" % (rk[a:b].mean(), rk[a:b].max()),
                  "zr %.1f" % zr[a:b].mean(), "nsig %.1f/%d" % (ns[a:b].mean(), ns[a:b].max()))

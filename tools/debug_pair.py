"""Inspect the row total weight Zhat of one pair (debugging aid): python tools/debug_pair.py P7"""
import sys, os
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
from oracle.structure import DH2Structure
name = sys.argv[1]
cfg = get_config(name); xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
try:
    h.recompress(cfg["eps"])
except Exception as e:
    print("recompress failed:", e)
k = h.k
rp = h.export("row_pairs", np.int64).reshape(-1, 3)
zoff = h.export("Z_off_row", np.int64); zr = h.export("Z_rows_row", np.int32)
Z = h.export("Z_row", np.complex128)
par_bad = []
for p in range(len(rp)):
    if zoff[p] < 0: continue
    z = Z[zoff[p]:zoff[p] + zr[p] * k]
    if not np.all(np.isfinite(z)):
        zz = z.reshape(k, zr[p]).T
        badr = np.where(~np.all(np.isfinite(zz), axis=1))[0]; badc = np.where(~np.all(np.isfinite(zz), axis=0))[0]
        par_bad.append(p)
        if len(par_bad) <= 3:
            print("pair", p, tuple(rp[p]), "zr", zr[p], "bad rows", badr[:8], "n", len(badr), "bad cols", badc[:8], "n", len(badc))
            print("   finite part max |.| %.3e" % np.nanmax(np.abs(zz[np.isfinite(zz)])))
print("bad pairs", len(par_bad))
blocks = h.export("blocks", np.int64).reshape(-1, 3); omega = h.export("omega", np.float64); g2 = h.export("normG2", np.float64)
bp = h.export("basis_pairs", np.int64).reshape(-1, 3); bpid = {(int(t), int(c)): i for i, (_, t, c) in enumerate(bp)}
VR = h.export("VR", np.complex128); roff = h.export("bp_R_off", np.int64); rr = h.export("bp_R_rows", np.int32)
S = h.export("S", np.complex128)
for p in par_bad[:2]:
    _, t, c = rp[p]
    for b in np.where((blocks[:, 0] == t) & (blocks[:, 2] == c))[0]:
        s = int(blocks[b, 1]); i = bpid[(s, int(c))]
        R = VR[roff[i]:roff[i] + rr[i] * k]
        Sb = S[b * k * k:(b + 1) * k * k]
        print("  block", b, "s", s, "omega %.3e normG2 %.3e" % (omega[b], g2[b]), "R finite", np.all(np.isfinite(R)), "R max %.2e" % np.abs(R).max(),
              "S finite", np.all(np.isfinite(Sb)), "S max %.2e min %.2e" % (np.abs(Sb).max(), np.abs(Sb).min()))

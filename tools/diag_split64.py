"""Diagnostic: where do the sigma exports of truncate_split64 = 1 / 0 differ (C4s)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import get_config, mesh_for, seeded_vector
from paper_1809_04384_b200 import DH2
name = sys.argv[1] if len(sys.argv) > 1 else "C4s"
cfg = get_config(name)
xyz, tri = mesh_for(cfg)
out = []
for v in (1, 0):
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    h.set_option("truncate_split64", v)
    h.set_option("truncate_split64_inner", v)
    h.recompress(cfg["eps"])
    x = seeded_vector(h.n, 3)
    out.append(dict(rank=h.export("rank_row", np.int32), sig=h.export("sigma_row", np.float64),
                    nsig=h.export("nsig_row", np.int32), off=h.export("sig_off_row", np.int64),
                    y=h.matvec(x, 1), lev=h.export("lev_ptr_row", np.int32) if True else None))
    h.close()
a, b = out
print("ranks equal", np.array_equal(a["rank"], b["rank"]), "nsig equal", np.array_equal(a["nsig"], b["nsig"]))
print("matvec equal", np.array_equal(a["y"], b["y"]), np.abs(a["y"] - b["y"]).max() / np.abs(a["y"]).max())
bad = np.nonzero(a["sig"] != b["sig"])[0]
print("sigma differ at", len(bad), "of", len(a["sig"]))
off = a["off"]
pairs = np.searchsorted(off, bad, side="right") - 1
lev = a["lev"]
valid = 0
for p in np.unique(pairs)[:20]:
    idx = bad[pairs == p] - off[p]
    inval = idx < a["nsig"][p]
    valid += inval.sum()
    print("pair", p, "level idx", np.searchsorted(lev, p, side="right") - 1, "nsig", a["nsig"][p], b["nsig"][p],
          "rank", a["rank"][p], "bad slots", idx[:8], "within nsig", inval.sum())
print("bad pairs", len(np.unique(pairs)), "levels", np.unique(np.searchsorted(lev, np.unique(pairs), side="right") - 1))

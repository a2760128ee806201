"""List pairs whose GPU singular values disagree with the oracle (debug helper)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
from conftest import oracle_run
from gpu_view import GpuView
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
name = sys.argv[1] if len(sys.argv) > 1 else "P1"
cfg = get_config(name); xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"]); h.recompress(cfg["eps"])
rc = oracle_run(name)
g = GpuView(h, rc.st)
sw = h.export("sweeps_row", np.int32)
keys = [(int(t), int(c)) for _, t, c in h.export("row_pairs", np.int64).reshape(-1, 3)]
bad = 0
for p, key in enumerate(keys):
    so, sg = rc.row.sigma[key], g.row.sigma[key]
    n = min(len(so), len(sg))
    err = np.abs(so[:n] - sg[:n]).max(initial=0) / max(so[0] if len(so) else 1, 1e-300)
    if err > 1e-12:
        bad += 1
        if bad < 12:
            ct = rc.st.ct
            leaf = ct.is_leaf(key[0])
            rows = ct.size(key[0]) if leaf else sum(rc.row.rank[(int(ch), rc.st.sd(int(ct.level[key[0]]), key[1]))] for ch in ct.children[key[0]])
            print(key, "leaf" if leaf else "inner", "rowsM", rows, "zr", rc.row.Zhat[key].shape[0], "nsig gpu/orc", len(sg), len(so), "sweeps", sw[p], "err %.2e" % err)
print("bad pairs", bad, "of", len(keys))

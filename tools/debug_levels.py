"""Per-level invariant errors of the GPU results against the oracle (debugging aid):
python tools/debug_levels.py P7 [truncate_workspace]"""
import sys, os
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
from conftest import oracle_run
from gpu_view import GpuView
name = sys.argv[1]
cfg = get_config(name); xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
if len(sys.argv) > 2: h.set_option("truncate_workspace", int(sys.argv[2]))
try:
    h.recompress(cfg["eps"])
except Exception as e:
    print("recompress failed:", e)
rc = oracle_run(name); st = rc.st; g = GpuView(h, st)
def rel(A, B):
    G0 = B.conj().T @ B; return np.abs(A.conj().T @ A - G0).max() / max(np.abs(G0).max(), 1e-300)
for l in st.active_levels:
    eR = max([rel(g.R(t, c), rc.R[(t, c)]) for (t, c) in st.basis_pairs[l]] or [0])
    eZ = max([rel(g.row.Zhat[(t, c)], rc.row.Zhat[(t, c)]) for (t, c) in st.row_pairs[l]] or [0])
    nanZ = sum(int(np.sum(~np.isfinite(g.row.Zhat[(t, c)]))) for (t, c) in st.row_pairs[l])
    rk = sum(int(g.row.rank[(t, c)] != rc.row.rank[(t, c)]) for (t, c) in st.row_pairs[l])
    print("level", l, "pairs", len(st.row_pairs[l]), "R err %.1e" % eR, "Z err %.1e" % eZ, "Z nonfinite", nanZ, "rank mismatches", rk, flush=True)
g2 = h.export("normG2", np.float64)
print("normG2 rel err %.1e" % np.max(np.abs(g2 - rc.normG ** 2) / rc.normG ** 2))
for nm in ("S", "E", "St"):
    a = h.export(nm, np.complex128)
    print(nm, "nonfinite", int(np.sum(~np.isfinite(a))), "of", a.size)
bad = [(t, c) for l in st.active_levels for (t, c) in st.row_pairs[l] if not np.all(np.isfinite(g.row.Zhat[(t, c)]))]
print("pairs with nonfinite Zhat:", len(bad))
for (t, c) in bad[:4]:
    Z = g.row.Zhat[(t, c)]
    rows = np.where(~np.all(np.isfinite(Z), axis=1))[0]; cols = np.where(~np.all(np.isfinite(Z), axis=0))[0]
    blks = [b for b in range(len(st.blocks)) if st.blocks[b][0] == t and st.blocks[b][2] == c]
    print((t, c), "Z shape", Z.shape, "bad rows", rows[:10], "bad cols", cols[:10], "blocks", [(int(st.blocks[b][1]), float(rc.omega[b])) for b in blks],
          "parents", [(tp, cp) for (tp, cp) in rc.row.Zhat if tp == st.ct.parent[t]][:4] if hasattr(st.ct, "parent") else "")

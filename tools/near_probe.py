"""Nearfield assembly + 3 nearfield matvecs on one config (for ncu captures of k_near_* / k_mv_near)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth import get_config, mesh_for, seeded_vector  # noqa: E402
from paper_1809_04384_b200 import DH2  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
h.set_profiling(True)
h.nearfield_assemble()
x = seeded_vector(h.n, 1)
for _ in range(3):
    h.matvec(x, 0, add_near=True)
s = h.stats()
print({k: s["kernels"][k] for k in ("nearfield", "matvec_near")}, s["nearfield"])
h.close()

"""Nearfield assembly + nearfield matvecs on one config (for ncu captures of k_near_* / k_mv_near*),
and the A/B of the two matvec forms (option near_tma).  usage: near_probe.py CONFIG [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth import get_config, mesh_for, seeded_vector  # noqa: E402
from paper_1809_04384_b200 import DH2  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = get_config(name)
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
h.recompress(cfg["eps"])  # the lean plan (C4/C5) has no ORIG matvec
h.set_profiling(True)
h.nearfield_assemble()
x = seeded_vector(h.n, 1)
prev = dict(ms=0.0, bytes=0.0, launches=0)
ys = {}
for tma in (0, 1, 0, 1):
    h.set_option("near_tma", tma)
    for _ in range(reps):
        ys[tma] = h.matvec(x, 1, add_near=True)
    k = h.stats()["kernels"]["matvec_near"]
    ms = (k["ms"] - prev["ms"]) / (k["launches"] - prev["launches"])
    gb = (k["bytes"] - prev["bytes"]) / (k["launches"] - prev["launches"]) / 1e9
    print("near_tma=%d: %.4f ms per launch, %.3f GB, %.0f GB/s" % (tma, ms, gb, gb / ms * 1e3))
    prev = dict(k)
print("rel diff tma vs direct: %.2e" % (np.linalg.norm(ys[1] - ys[0]) / np.linalg.norm(ys[0])))
s = h.stats()
print({k: s["kernels"][k] for k in ("nearfield", "matvec_near")}, s["nearfield"])
h.close()

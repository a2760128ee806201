"""A/B of the far-field matvec launch shapes (option mv_forward_warp) after a recompression.
usage: mv_probe.py CONFIG [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from synth import get_config, mesh_for, seeded_vector  # noqa: E402
from paper_1809_04384_b200 import DH2  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = get_config(name)
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
h.recompress(cfg["eps"])
h.set_profiling(True)
x = seeded_vector(h.n, 1)
h.matvec(x, 1)
prev = dict(h.stats()["kernels"]["matvec"])
ys = {}
for v in (0, 1, 2, 0, 1, 2):
    h.set_option("mv_forward_warp", v)
    for _ in range(reps):
        ys[v] = h.matvec(x, 1)
    k = h.stats()["kernels"]["matvec"]
    ms = (k["ms"] - prev["ms"]) / reps
    gb = (k["bytes"] - prev["bytes"]) / reps / 1e9
    print("mv_forward_warp=%d: %.3f ms per matvec, %.2f GB, %.0f GB/s" % (v, ms, gb, gb / ms * 1e3 if ms else 0))
    prev = dict(k)
for v in (1, 2):
    print("rel diff %d vs 0: %.2e" % (v, np.linalg.norm(ys[v] - ys[0]) / np.linalg.norm(ys[0])))
h.close()

"""A/B of the leaf truncation variants on C4/C5 (lean plan): fuse_leaf_weights 0 / 2, recompress
time and the top kernel classes.  usage: python tools/fuse_probe.py [C4 C5]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_04384_b200 import DH2  # noqa: E402
from synth import get_config, mesh_for  # noqa: E402

for name in (sys.argv[1:] or ["C4", "C5"]):
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    for fuse in (0, 2, 0, 2):
        h.set_option("fuse_leaf_weights", fuse)
        h.set_profiling(True)
        s0 = h.stats()["kernels"]
        t = time.time()
        h.recompress(cfg["eps"])
        dt = time.time() - t
        s1 = h.stats()
        ks = {k: round(v["ms"] - s0.get(k, {"ms": 0})["ms"], 1) for k, v in s1["kernels"].items()}
        top = dict(sorted(ks.items(), key=lambda kv: -kv[1])[:8])
        print(name, "fuse", fuse, "recompress %.3f s" % dt, "E_row %.6e" % s1["E_row"], top, flush=True)
    h.close()

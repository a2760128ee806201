"""A/B of a dh2_set_option on C4/C5 (lean plan): recompress time and top kernel classes per value.
usage: python tools/ab_probe.py OPTION V0,V1[,V2...] [configs...]  (each value run twice, interleaved)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_04384_b200 import DH2  # noqa: E402
from synth import get_config, mesh_for  # noqa: E402

opt, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
for name in (sys.argv[3:] or ["C4", "C5"]):
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    for v in vals + vals:
        h.set_option(opt, v)
        h.set_profiling(True)
        s0 = h.stats()["kernels"]
        t = time.time()
        h.recompress(cfg["eps"])
        dt = time.time() - t
        s1 = h.stats()
        ks = {k: round(x["ms"] - s0.get(k, {"ms": 0})["ms"], 1) for k, x in s1["kernels"].items()}
        print(name, opt, v, "recompress %.3f s" % dt, "E_row %.9e" % s1["E_row"], dict(sorted(ks.items(), key=lambda kv: -kv[1])[:8]),
              flush=True)
    h.close()

"""One recompression with dh2_set_option values (profiling target for ncu).
usage: python tools/opt_probe.py CONFIG [option=value ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_04384_b200 import DH2  # noqa: E402
from synth import get_config, mesh_for  # noqa: E402

cfg = get_config(sys.argv[1])
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    h.set_option(k, int(v))
h.set_profiling(True)
t = time.time()
h.recompress(cfg["eps"])
s = h.stats()
print(sys.argv[1:], "recompress %.3f s" % (time.time() - t), "E_row %.9e" % s["E_row"],
      dict(sorted(((k, round(x["ms"], 1)) for k, x in s["kernels"].items()), key=lambda kv: -kv[1])[:10]))
h.close()

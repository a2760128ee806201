"""Wall-clock breakdown of one end-to-end call sequence through the C ABI (host buffers)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for, seeded_vector
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
xyz, tri = mesh_for(cfg)
x = seeded_vector(tri.shape[0], 2)
for it in range(3):
    t0 = time.perf_counter()
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    t1 = time.perf_counter()
    h.recompress(cfg["eps"])
    t2 = time.perf_counter()
    y = h.matvec(x, 1)
    t3 = time.perf_counter()
    s = h.stats()
    h.close()
    t4 = time.perf_counter()
    print("iter %d build %.1f ms (host structure %.1f ms) recompress %.1f ms matvec %.1f ms destroy %.1f ms total %.1f ms"
          % (it, 1e3 * (t1 - t0), s["host_build_ms"], 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t4 - t0)))
    print("   host phases ms", {k: round(v, 2) if isinstance(v, float) else v for k, v in s["host_phases_ms"].items()})

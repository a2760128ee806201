"""Fresh-context vs warm recompression: host wall clock per lean phase and device kernel time
(where do the extra seconds of the end-to-end call go?)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import get_config, mesh_for  # noqa: E402
from paper_1809_04384_b200 import DH2  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
xyz, tri = mesh_for(cfg)
for it in range(2):
    t0 = time.perf_counter()
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    h.set_profiling(True)
    t1 = time.perf_counter()
    for rep in range(2):
        k0 = h.stats()["kernels"]
        ta = time.perf_counter()
        h.recompress(cfg["eps"])
        tb = time.perf_counter()
        s = h.stats()
        dev = sum(v["ms"] - k0.get(k, {}).get("ms", 0.0) for k, v in s["kernels"].items())
        print("ctx %d rep %d: build %.0f ms, recompress wall %.0f ms, device kernels %.0f ms, lean wall %s" %
              (it, rep, 1e3 * (t1 - t0), 1e3 * (tb - ta), dev,
               {k: round(v) for k, v in s["lean"].get("wall_ms", {}).items()}), flush=True)
    t2 = time.perf_counter()
    h.close()
    print("   close %.0f ms" % (1e3 * (time.perf_counter() - t2)), flush=True)

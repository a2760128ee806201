"""Build + recompress one configuration (auto plan: full if it fits, else memory-lean), print the
plan, per-phase device times and memory.  usage: python tools/lean_probe.py C4 [chunks]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_04384_b200 import DH2  # noqa: E402
from synth import get_config, mesh_for, seeded_vector  # noqa: E402

name = sys.argv[1]
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = get_config(name)
xyz, tri = mesh_for(cfg)
t0 = time.time()
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
t1 = time.time()
if chunks:
    h.set_option("lean_chunks", chunks)
h.set_profiling(True)
for it in range(2):
    t2 = time.time()
    h.recompress(cfg["eps"])
    t3 = time.time()
    print("recompress %d: %.3f s" % (it, t3 - t2), flush=True)
x = seeded_vector(h.n, 1)
y = h.matvec(x, 1)
t4 = time.time()
s = h.stats()
sw = h.export("sweeps_row", np.int32)
lp = h.export("lev_ptr_row", np.int32)
sweeps = {int(l): np.bincount(sw[lp[l]:lp[l + 1]]).tolist() for l in range(len(lp) - 1) if lp[l + 1] > lp[l]}
ks = {k: round(v["ms"], 1) for k, v in sorted(s["kernels"].items(), key=lambda kv: -kv[1]["ms"])[:25]}
print(json.dumps({"config": name, "build_s": t1 - t0, "matvec_s": t4 - t3, "lean": s["lean"], "device_bytes": s["device_bytes"],
                  "storage": h.storage(1), "E_row": s["E_row"], "far2": s["far2"], "ynorm": float(np.linalg.norm(y)),
                  "kernels_ms_2runs": ks, "jacobi_sweeps_hist_per_level": sweeps}), flush=True)

"""Per-level rank statistics of a recompressed configuration (sizing of the memory-lean plan).
usage: python tools/rank_stats.py C4q [C5q ...]"""
import json
import sys
import os
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_04384_b200 import DH2  # noqa: E402
from synth import get_config, mesh_for  # noqa: E402

for name in sys.argv[1:]:
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    t0 = time.time()
    h.recompress(cfg["eps"])
    dt = time.time() - t0
    rank = h.export("rank_row", np.int32)
    lp = h.export("lev_ptr_row", np.int32)
    ch0 = h.export("child0_row", np.int32)
    out = {"config": name, "recompress_s": dt, "storage": h.storage(1), "levels": {}}
    for l in range(len(lp) - 1):
        a, b = lp[l], lp[l + 1]
        if b <= a:
            continue
        r = rank[a:b]
        out["levels"][l] = {"pairs": int(b - a), "mean": float(r.mean()), "max": int(r.max()),
                            "p90": float(np.percentile(r, 90)), "leaf": bool(ch0[a] < 0)}
    print(json.dumps(out), flush=True)
    h.close()

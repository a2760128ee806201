"""Run one configuration through the C ABI (debugging aid; DH2_DEBUG_SYNC=1 names the failing kernel):
python tools/debug_cfg.py C5s [truncate_workspace]   or   python tools/debug_cfg.py cube:16:14:5:64:1e-6"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
if ":" in sys.argv[1]:
    mesh, q, kappa, m, leaf, eps = sys.argv[1].split(":")
    cfg = dict(mesh=mesh, q=int(q), kappa=float(kappa), m=int(m), leaf=int(leaf), eta1=1.0, eta2=10.0, eps=float(eps))
else:
    cfg = get_config(sys.argv[1])
xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
if len(sys.argv) > 2:
    h.set_option("truncate_workspace", int(sys.argv[2]))
print("built", sys.argv[1:], flush=True)
h.set_profiling(True)
h.recompress(cfg["eps"])
s = h.stats()
print("ok", s["truncate_ws_launches"], {k: v["launches"] for k, v in s["kernels"].items()}, flush=True)

mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lean.py -x -q -k "truncate_paths or lean" > gpurun_out/pytest_r2l.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r2l.log
cat > /tmp/fuseprobe.py <<'PY'
import sys, json, time
sys.path.insert(0, '.')
import numpy as np
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
for name in ("C4", "C5"):
    cfg = get_config(name); xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    for fuse in (0, 2, 0, 2):
        h.set_option("fuse_leaf_weights", fuse)
        h.set_profiling(True)
        s0 = h.stats()["kernels"]
        t = time.time(); h.recompress(cfg["eps"]); dt = time.time() - t
        s1 = h.stats()
        ks = {k: round(v["ms"] - s0.get(k, {"ms": 0})["ms"], 1) for k, v in s1["kernels"].items()}
        top = dict(sorted(ks.items(), key=lambda kv: -kv[1])[:8])
        print(name, "fuse", fuse, "recompress %.3f s" % dt, "E_row %.6e" % s1["E_row"], top, flush=True)
    h.close()
PY
timeout 900 python /tmp/fuseprobe.py > gpurun_out/fuseprobe.log 2>&1; echo "fuse rc=$?"; cat gpurun_out/fuseprobe.log

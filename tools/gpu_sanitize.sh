# compute-sanitizer, ONE tool per gpurun call: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck
mkdir -p gpurun_out
T=${1:-memcheck}
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
cat > /tmp/san.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for, seeded_vector
for name, chunks, world in (("P1", 0, 1), ("P8", 0, 1), ("P4", 0, 1), ("P2", 3, 1), ("P1", 0, 2), ("C1", 2, 2)):
    cfg = get_config(name); xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], world=world)
    if chunks:
        h.set_option("lean_chunks", chunks)
    h.recompress(cfg["eps"])
    y = h.matvec(seeded_vector(h.n, 1), 1)
    if not chunks:
        y0 = h.matvec(seeded_vector(h.n, 1), 0)
    print(name, chunks, world, "ok", float(np.linalg.norm(y)), flush=True)
    h.close()
PY
timeout 2400 compute-sanitizer --tool $T --error-exitcode 7 --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_$T.log 2>&1; echo "sanitizer $T rc=$?"; tail -15 gpurun_out/sanitize_$T.log

mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_device_blocks.py -x -q -k append > gpurun_out/pytest_r2s_dev.log 2>&1; echo "dev rc=$?"; tail -3 gpurun_out/pytest_r2s_dev.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "column_by_column" > gpurun_out/pytest_r2s.log 2>&1; echo "par rc=$?"; tail -3 gpurun_out/pytest_r2s.log
cat > /tmp/flagprobe.py <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_1809_04384_b200 import DH2
from synth import get_config, mesh_for
cfg = get_config("C4"); xyz, tri = mesh_for(cfg)
h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
for flag in (0, 1, 0, 1):
    h.set_option("qr_flag", flag); h.set_profiling(True)
    s0 = h.stats()["kernels"]; t = time.time(); h.recompress(cfg["eps"]); dt = time.time() - t
    s1 = h.stats(); ks = {k: round(v["ms"] - s0.get(k, {"ms": 0})["ms"], 1) for k, v in s1["kernels"].items()}
    print("flag", flag, "recompress %.3f s" % dt, "E_row %.9e" % s1["E_row"], dict(sorted(ks.items(), key=lambda kv: -kv[1])[:8]), flush=True)
PY
timeout 600 python /tmp/flagprobe.py > gpurun_out/flagprobe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/flagprobe.log

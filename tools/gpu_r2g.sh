# WY appends: device unit test, k=125 parity, lean bitwise, then scale parity and a C4 A/B
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_device_blocks.py -x -q -k append > gpurun_out/pytest_r2g_dev.log 2>&1; echo "devtest rc=$?"; tail -3 gpurun_out/pytest_r2g_dev.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lean.py -x -q -k "P4 or P5 or P6 or P7 or C4s or column_by_column" > gpurun_out/pytest_r2g_par.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_r2g_par.log
timeout 600 python tools/lean_probe.py C4 > gpurun_out/probe_c4_wy.log 2>&1; echo "probe rc=$?"; tail -1 gpurun_out/probe_c4_wy.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('kernels_ms_2runs',)})"
grep recompress gpurun_out/probe_c4_wy.log
timeout 2400 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity_sampled.py -x -q --durations=10 > gpurun_out/pytest_r2g_scale.log 2>&1; echo "scale rc=$?"; tail -15 gpurun_out/pytest_r2g_scale.log

mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 600 python tools/lean_probe.py C4 > gpurun_out/probe_c4_k.log 2>&1; echo "probe rc=$?"; grep recompress gpurun_out/probe_c4_k.log; tail -1 gpurun_out/probe_c4_k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms_2runs']); print(d['jacobi_sweeps_hist_per_level'])"
timeout 3000 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_r2k.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_r2k.log

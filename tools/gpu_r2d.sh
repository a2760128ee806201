mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 1200 python -m pytest tests/test_gpu_lean.py -x -q > gpurun_out/pytest_lean.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_lean.log
timeout 600 python tools/lean_probe.py C4q 4 > gpurun_out/probe_c4q.log 2>&1; echo "probe c4q rc=$?"; tail -4 gpurun_out/probe_c4q.log

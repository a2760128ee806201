mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_lean.py -x -q > gpurun_out/pytest_r2j_lean.log 2>&1; echo "lean rc=$?"; tail -5 gpurun_out/pytest_r2j_lean.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_r2j.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_r2j.log

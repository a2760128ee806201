mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 3600 python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/pytest_r2q.log 2>&1; echo "pytest rc=$?"; tail -18 gpurun_out/pytest_r2q.log

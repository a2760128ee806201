# round 2, call A: FP64 peaks + new parity tests (storage, G5 at C2)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 300 python tools/fp64_peak.py --out gpurun_out/fp64_peak.json > gpurun_out/fp64_peak.log 2>&1; echo "peak rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -k "storage or G5" > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2a.log

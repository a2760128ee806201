mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lean.py -x -q -k "G3 or G4 or truncate_paths or lean" > gpurun_out/pytest_r2m.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2m.log
timeout 900 python tools/fuse_probe.py > gpurun_out/fuseprobe_m.log 2>&1; echo "fuse rc=$?"; cat gpurun_out/fuseprobe_m.log

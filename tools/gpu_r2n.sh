mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 900 python tools/fuse_probe.py > gpurun_out/fuseprobe_n.log 2>&1; echo "fuse rc=$?"; cat gpurun_out/fuseprobe_n.log
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_lean.py tests/test_gpu_nccl.py -x -q > gpurun_out/pytest_r2n.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2n.log

mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 900 python tools/lean_probe.py C4 > gpurun_out/probe_c4.log 2>&1; echo "probe c4 rc=$?"; tail -4 gpurun_out/probe_c4.log
timeout 900 python tools/lean_probe.py C5 > gpurun_out/probe_c5.log 2>&1; echo "probe c5 rc=$?"; tail -4 gpurun_out/probe_c5.log

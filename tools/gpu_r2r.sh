mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 600 python tools/lean_probe.py C4 > gpurun_out/probe_c4_r.log 2>&1; echo "probe rc=$?"; grep recompress gpurun_out/probe_c4_r.log; tail -1 gpurun_out/probe_c4_r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels_ms_2runs'], d['E_row'])"
timeout 2400 python -m pytest tests/test_gpu_device_blocks.py tests/test_gpu_parity.py tests/test_gpu_lean.py tests/test_gpu_parity_scale.py -x -q -k "append or P4 or P5 or P7 or C2 or lean or scale" > gpurun_out/pytest_r2r.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_r2r.log

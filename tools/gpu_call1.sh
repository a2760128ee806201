# verification of HEAD + r02g profiles (usage: gpurun -- 'bash tools/gpu_call1.sh')
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_nearfield.py tests/test_gpu_lean.py -m gpu -x -q > gpurun_out/r02g_pytest_near_lean.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/near_probe.py C4 > gpurun_out/r02g_near_probe_c4.log 2>&1; echo "near probe rc=$?"
bash tools/gpu_profile_r02g.sh

mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nearfield.py -m gpu -x -q -k "tma or full_matvec or shards" > gpurun_out/r02h_pytest_new.log 2>&1; echo "new tests rc=$?"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "G1" > gpurun_out/r02h_pytest_g1.log 2>&1; echo "G1 rc=$?"
timeout 600 python tools/near_probe.py C4 > gpurun_out/r02h_near_probe_c4.log 2>&1; echo "near probe C4 rc=$?"
timeout 300 python tools/near_probe.py C3 > gpurun_out/r02h_near_probe_c3.log 2>&1
timeout 300 python tools/near_probe.py C2 > gpurun_out/r02h_near_probe_c2.log 2>&1
timeout 600 python tools/lean_probe.py C4 > gpurun_out/r02h_lean_probe_c4.log 2>&1

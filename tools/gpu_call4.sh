mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r02j_bench_c4.json 2> gpurun_out/r02j_bench_c4.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_lean.py tests/test_gpu_nearfield.py tests/test_gpu_parity_scale.py -m gpu -q -k "G4 or matvec or shard or lean or scale" > gpurun_out/r02j_pytest_matvec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02j_pytest_matvec.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02j_bench_c3.json 2> gpurun_out/r02j_bench_c3.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/r02j_bench_c2.json 2> gpurun_out/r02j_bench_c2.err

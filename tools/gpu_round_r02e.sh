# round-2 evidence after the nearfield (usage: gpurun -- 'bash tools/gpu_round_r02e.sh')
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
timeout 600 python tools/near_probe.py C3 > gpurun_out/near_probe_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_near|k_mv_near" -c 3 -o gpurun_out/near_c3 python tools/near_probe.py C3 > gpurun_out/ncu_near.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err

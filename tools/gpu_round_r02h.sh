# final round-2 evidence on one B200 (usage: gpurun -- 'bash tools/gpu_round_r02h.sh'): new tests first,
# A/B of the nearfield matvec forms, the default bench line (C4), full GPU tests, the other configs,
# the reference arm, the launch list of the bench command and two full captures (k_mv_near_tma, k_leafV)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02h_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_nearfield.py -m gpu -x -q -k "tma or full_matvec or shards" > gpurun_out/r02h_pytest_new.log 2>&1; echo "new tests rc=$?"
timeout 600 python tools/near_probe.py C4 > gpurun_out/r02h_near_probe_c4.log 2>&1; echo "near probe C4 rc=$?"
timeout 300 python tools/near_probe.py C3 > gpurun_out/r02h_near_probe_c3.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r02h_bench_c4.json 2> gpurun_out/r02h_bench_c4.err; echo "bench rc=$?"
timeout 3600 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_pytest_gpu.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02h_bench_c5.json 2> gpurun_out/r02h_bench_c5.err
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/r02h_bench_c3.json 2> gpurun_out/r02h_bench_c3.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r02h_bench_c2.json 2> gpurun_out/r02h_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02h_bench_ref.json 2> gpurun_out/r02h_bench_ref.err
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_c4.csv $B > gpurun_out/ncu_r02h_launch.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py launches gpurun_out/r02h_launches_c4.csv > gpurun_out/r02h_launches_c4.md 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mv_near_tma" -s 2 -c 1 -o /tmp/r02h_k_mv_near_tma python tools/near_probe.py C4 3 > gpurun_out/ncu_r02h_near.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leafV" -s 3 -c 1 -o /tmp/r02h_k_leafV python tools/lean_probe.py C4 > gpurun_out/ncu_r02h_leafV.log 2>&1
for k in k_mv_near_tma k_leafV; do
  python tools/ncu_summary.py full /tmp/r02h_$k.ncu-rep | tail -1 >> gpurun_out/r02h_kernels.md
  ncu -i /tmp/r02h_$k.ncu-rep --page raw --csv > gpurun_out/r02h_raw_$k.csv 2>/dev/null
done
ls -la gpurun_out/

# final round-2 evidence on one B200 (usage: gpurun -- 'bash tools/gpu_round_r02i.sh'): the new tests first,
# A/B probes of the nearfield and far-field matvec forms, the default bench line (C4), the launch list of the
# bench command, two full captures, the other configs, the reference arm, then the full GPU test suite
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02i_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_nearfield.py tests/test_gpu_parity.py -m gpu -q -k "tma or full_matvec or shards or blocks_all or G4" > gpurun_out/r02i_pytest_new.log 2>&1; echo "new tests rc=$?"
timeout 600 python tools/mv_probe.py C4 > gpurun_out/r02i_mv_probe_c4.log 2>&1; echo "mv probe C4 rc=$?"
timeout 300 python tools/mv_probe.py C3 > gpurun_out/r02i_mv_probe_c3.log 2>&1
timeout 300 python tools/mv_probe.py C2 20 > gpurun_out/r02i_mv_probe_c2.log 2>&1
timeout 600 python tools/near_probe.py C4 > gpurun_out/r02i_near_probe_c4.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r02i_bench_c4.json 2> gpurun_out/r02i_bench_c4.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches_c4.csv $B > gpurun_out/ncu_r02i_launch.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py launches gpurun_out/r02i_launches_c4.csv > gpurun_out/r02i_launches_c4.md 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mv_near_tma" -s 2 -c 1 -o /tmp/r02i_k_mv_near_tma python tools/near_probe.py C4 3 > gpurun_out/ncu_r02i_near.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mv_forward" -s 10 -c 1 -o /tmp/r02i_k_mv_forward python tools/mv_probe.py C4 1 > gpurun_out/ncu_r02i_fwd.log 2>&1
for k in k_mv_near_tma k_mv_forward; do
  python tools/ncu_summary.py full /tmp/r02i_$k.ncu-rep | tail -1 >> gpurun_out/r02i_kernels.md
  ncu -i /tmp/r02i_$k.ncu-rep --page raw --csv > gpurun_out/r02i_raw_$k.csv 2>/dev/null
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02i_bench_c5.json 2> gpurun_out/r02i_bench_c5.err
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/r02i_bench_c3.json 2> gpurun_out/r02i_bench_c3.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r02i_bench_c2.json 2> gpurun_out/r02i_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02i_bench_ref.json 2> gpurun_out/r02i_bench_ref.err
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest_gpu.log
ls -la gpurun_out/

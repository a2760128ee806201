# round-2 final evidence on one B200 (usage: gpurun -- 'bash tools/gpu_round_r02d.sh'): GPU tests,
# smoke, bench lines (C4 default with e2e and the oracle baseline, C5, C3, C2, the reference arm),
# the C4 launch list and full ncu captures of the top kernels (summaries written on the box).
set -x
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2d_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2d_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r2d_bench_c4.json 2> gpurun_out/r2d_bench_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2d_bench_c5.json 2> gpurun_out/r2d_bench_c5.err
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/r2d_bench_c3.json 2> gpurun_out/r2d_bench_c3.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r2d_bench_c2.json 2> gpurun_out/r2d_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2d_bench_ref.json 2> gpurun_out/r2d_bench_ref.err
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_c4.csv $B > gpurun_out/r2d_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py launches gpurun_out/r2d_launches_c4.csv > gpurun_out/r2d_launches_c4.md 2>&1
P="python tools/lean_probe.py C4"
for k in k_trunc_jepi64 k_trunc_qr64 k_basis_cq k_total_weights_cq k_block_weights; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 0 -c 1 -o /tmp/r2d_$k $P > gpurun_out/r2d_ncu_$k.log 2>&1
  echo "$k rc=$?"
  python tools/ncu_summary.py full /tmp/r2d_$k.ncu-rep | tail -1 >> gpurun_out/r2d_kernels_c4.md
  python tools/ncu_lines.py /tmp/r2d_$k.ncu-rep 40 > gpurun_out/r2d_lines_c4_$k.txt
  ncu -i /tmp/r2d_$k.ncu-rep --page raw --csv > gpurun_out/r2d_raw_$k.csv 2>/dev/null
done
ls -la gpurun_out/ | grep r2d

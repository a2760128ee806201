# round-2 final profiles of the bench command (usage: gpurun -- 'bash tools/gpu_profile_r02g.sh')
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B > gpurun_out/plain_bench_g.json 2> gpurun_out/plain_bench_g.err; echo "plain bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_launches_c4.csv $B > gpurun_out/ncu_r02g_launch.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py launches gpurun_out/r02g_launches_c4.csv > gpurun_out/r02g_launches_c4.md 2>&1
P="python tools/lean_probe.py C4"
for spec in "k_trunc_jepi64:0" "k_trunc_qr64:0" "k_basis_cq:1" "k_total_weights_cq:0" "k_block_weights:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 -o /tmp/r02g_$k $P > gpurun_out/ncu_r02g_$k.log 2>&1
  echo "$k rc=$?"
  python tools/ncu_summary.py full /tmp/r02g_$k.ncu-rep | tail -1 >> gpurun_out/r02g_kernels.md
  python tools/ncu_lines.py /tmp/r02g_$k.ncu-rep 40 > gpurun_out/r02g_lines_$k.txt
  ncu -i /tmp/r02g_$k.ncu-rep --page raw --csv > gpurun_out/r02g_raw_$k.csv 2>/dev/null
done
python tools/pairstats.py C4 > gpurun_out/r02g_pairstats_c4.log 2>&1
ls -la gpurun_out/

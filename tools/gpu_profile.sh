# round-2 profiles (retry, summaries made on the box; the reports themselves exceed the copy-back limit)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B > gpurun_out/plain_bench_p.log 2>&1; echo "plain bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_launches_c4.csv $B > gpurun_out/ncu_r2p_launch.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py launches gpurun_out/r2p_launches_c4.csv > gpurun_out/r2p_launches_c4.md 2>&1
P="python tools/lean_probe.py C4"
$P > gpurun_out/plain_probe_p.log 2>&1; echo "plain probe rc=$?"
for spec in "k_basis:1" "k_total_weights:4" "k_truncate:0" "k_block_weights:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s $s -c 1 -o /tmp/r2p_$k $P > gpurun_out/ncu_r2p_$k.log 2>&1
  echo "$k rc=$?"
  python tools/ncu_summary.py full /tmp/r2p_$k.ncu-rep | tail -1 >> gpurun_out/r2p_kernels.md
  python tools/ncu_lines.py /tmp/r2p_$k.ncu-rep 40 > gpurun_out/r2p_lines_$k.txt
  ncu -i /tmp/r2p_$k.ncu-rep --page raw --csv > gpurun_out/r2p_raw_$k.csv 2>/dev/null
done
ls -la gpurun_out/

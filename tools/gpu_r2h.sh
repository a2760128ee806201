# ncu: full captures of the three main k=125 kernels (C4q, lean plan, 4 chunks) + launch list of one C4 bench step
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
P="python tools/lean_probe.py C4q 4"
$P > gpurun_out/plain_probe.log 2>&1; echo "plain rc=$?"
for spec in "k_basis:0" "k_total_weights:3" "k_truncate:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s $s -c 1 -o gpurun_out/r2h_$k $P > gpurun_out/ncu_r2h_$k.log 2>&1
  echo "$k rc=$?"
done
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B > gpurun_out/plain_bench.log 2>&1; echo "plain bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_c4.csv $B > gpurun_out/ncu_r2h_launch.log 2>&1; echo "launch list rc=$?"
for f in gpurun_out/r2h_k_*.ncu-rep; do python tools/ncu_summary.py full $f | tail -1; done > gpurun_out/r2h_kernels.md

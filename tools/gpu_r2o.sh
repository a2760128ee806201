# round-2 profiles: launch list of one C4 bench step + full captures of the main kernels at C4
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B > gpurun_out/plain_bench_o.log 2>&1; echo "plain bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_launches_c4.csv $B > gpurun_out/ncu_r2o_launch.log 2>&1; echo "launch list rc=$?"
P="python tools/lean_probe.py C4"
$P > gpurun_out/plain_probe_o.log 2>&1; echo "plain probe rc=$?"
# the chunk-0 launches: basis level 10 (2nd basis launch), total weights level 11 (5th), truncation level 11 (1st), block weights (1st)
for spec in "k_basis:1" "k_total_weights:4" "k_truncate:0" "k_block_weights:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s $s -c 1 -o gpurun_out/r2o_$k $P > gpurun_out/ncu_r2o_$k.log 2>&1
  echo "$k rc=$?"
done
for f in gpurun_out/r2o_k_*.ncu-rep; do python tools/ncu_summary.py full $f | tail -1; done > gpurun_out/r2o_kernels.md

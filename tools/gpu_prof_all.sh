# one ncu --set full capture per main kernel of a C2 step (the largest launch of each), for profiles/
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
for spec in "k_trunc_qr:0" "k_jacobi_w32:0" "k_trunc_epi:0" "k_total_weights:2" "k_basis:1" "k_block_weights:0" "k_leafV:0" "k_S:0" "k_project:0" "k_truncate:0" "k_mv_leaf_out:0"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s $s -c 1 -o gpurun_out/all_$k $B > /dev/null 2>&1
  echo "$k rc=$?"
done
# summaries only (the reports themselves exceed the copy-back limit)
for f in gpurun_out/all_*.ncu-rep; do python tools/ncu_summary.py full $f | tail -1; done > gpurun_out/all_kernels.md
for f in gpurun_out/all_*.ncu-rep; do ncu -i $f --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed 2>/dev/null | tail -1; done > gpurun_out/all_kernels_raw.csv
rm -f gpurun_out/all_*.ncu-rep

# full ncu captures of the main kernels of one C2 step + per-level pair statistics
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 300 python tools/pairstats.py C2 > gpurun_out/pairstats_c2.txt 2>&1
for spec in "k_basis:1" "k_total_weights:2" "k_block_weights:0" "k_leafV:0" "k_project:0" "k_truncate:1"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o gpurun_out/full_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done

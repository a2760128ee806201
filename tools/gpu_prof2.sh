mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 300 python tools/e2e_breakdown.py C2 > gpurun_out/e2e_c2.txt 2>&1
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_basis -s 1 -c 1 -o gpurun_out/basis3 $B > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_total_weights -s 2 -c 1 -o gpurun_out/tw3 $B > /dev/null 2>&1; echo "rc=$?"

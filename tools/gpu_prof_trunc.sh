mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_truncate -s 0 -c 1 -o gpurun_out/trunc2 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_t2.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_total_weights -s 2 -c 1 -o gpurun_out/tw2 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_tw2.log 2>&1; echo "ncu rc=$?"

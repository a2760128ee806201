# round 2: GPU suite (with lean + full-size C4/C5 sampled parity) + default bench (C4) + C2 bench
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_r2f.log
timeout 1500 python bench.py > gpurun_out/bench_r2f_c4.json 2> gpurun_out/bench_r2f_c4.err; echo "bench C4 rc=$?"
timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_r2f_c2.json 2> gpurun_out/bench_r2f_c2.err; echo "bench C2 rc=$?"

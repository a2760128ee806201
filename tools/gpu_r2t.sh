# round 2: full GPU suite + bench lines (default C4 with cpu baseline and e2e; C5, C3, C2)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 1500 python bench.py > gpurun_out/bench_t_c4.json 2> gpurun_out/bench_t_c4.err; echo "bench C4 rc=$?"; tail -c 600 gpurun_out/bench_t_c4.json
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_t_c5.json 2> gpurun_out/bench_t_c5.err; echo "bench C5 rc=$?"
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_t_c3.json 2> gpurun_out/bench_t_c3.err; echo "bench C3 rc=$?"
timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_t_c2.json 2> gpurun_out/bench_t_c2.err; echo "bench C2 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_t_ref.json 2> gpurun_out/bench_t_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_t_ref.json | tail -c 400
timeout 3600 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_t.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/pytest_t.log

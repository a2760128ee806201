mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 1500 python -m pytest tests/test_gpu_parity_sampled.py -m gpu -x -q > gpurun_out/pytest_sampled.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sampled.log
for c in C4s C5s C4q C5q; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done

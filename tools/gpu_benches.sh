# bench lines of the larger configurations (one GPU)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
for c in C4s C5s C4q C5q; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done

# round 2: full GPU suite + C2/C4q bench lines (no cpu baseline)
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2c.log
for c in C2 C4q; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_r2c_$c.json 2> gpurun_out/bench_r2c_$c.err; echo "bench $c rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_r2c_$c.json').read().strip().splitlines()[-1]); print('$c ms/step', d['ms_per_step'], {k:round(v['ms_per_step'],2) for k,v in d['phases'].items()})"; done

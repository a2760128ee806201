# build + a quick subset of GPU tests (arg 1: pytest -k expression, "" = none) + one bench line
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sub.log; fi
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'])
for k,v in sorted(d['launch_detail_ms_per_step'].items(), key=lambda kv:-kv[1])[:14]: print(' ', k, v)"

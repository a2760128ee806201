# quick GPU check: parity tests + one bench line (usage: bash tools/gpu_quick.sh [pytest -k expr])
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
K=${1:-}
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'])
for k,v in sorted(d['launch_detail_ms_per_step'].items(), key=lambda kv:-kv[1])[:12]: print(' ', k, v)"

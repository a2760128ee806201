bash tools/gpu_bench.sh "P0 or P1 or P2 or P3 or P4 or P5 or P6 or P7 or C1 or C2"
for c in C4q C5q; do timeout 600 python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c ms', d['ms_per_step']); print(sorted(d['launch_detail_ms_per_step'].items(), key=lambda kv:-kv[1])[:6])"; done

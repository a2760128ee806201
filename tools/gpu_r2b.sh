mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_1809_04384_b200 import build as b; b.build()"
(free -g; nproc; cat /sys/fs/cgroup/memory.max 2>/dev/null; lscpu | grep -i 'model name'; nvidia-smi --query-gpu=memory.total,memory.free --format=csv) > gpurun_out/box_info.txt 2>&1
timeout 900 python tools/rank_stats.py C4s C5s C4q C5q > gpurun_out/rank_stats.jsonl 2> gpurun_out/rank_stats.err; echo "rank rc=$?"

# A/B of the split-truncation Jacobi variants (arg 1: pytest -k expression, optional)
bash tools/gpu_bench.sh "${1:-}"
BENCH_ARGS="--option jacobi_two_warps=1" bash tools/gpu_bench.sh "" | grep -E "ms/step|truncate_row@8"

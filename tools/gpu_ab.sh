bash tools/gpu_bench.sh "P1 or C1" 2>&1 | grep -E "passed|failed|ms/step|truncate_row@8"
sed -i 's/__launch_bounds__(128, 4) k_jacobi_w32/__launch_bounds__(128, 3) k_jacobi_w32/' paper_1809_04384_b200/csrc/dh2_kernels.cu
bash tools/gpu_bench.sh "" 2>&1 | grep -E "ms/step|truncate_row@8"

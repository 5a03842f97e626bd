mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_gram_kernel|pair_var_kernel|mean_kernel|chol_panel" -c 4 -o gpurun_out/r01k_pair python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01k_ncu.out 2>&1

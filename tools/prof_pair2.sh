mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_var_kernel" -c 1 -o gpurun_out/r01n_var python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01n_ncu1.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_gram_kernel" -c 1 -o gpurun_out/r01n_gram python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01n_ncu2.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chol_panel" -s 5 -c 1 -o gpurun_out/r01n_chol python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01n_ncu3.out 2>&1

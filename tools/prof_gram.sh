mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -c 1 -o gpurun_out/r01f_gram_small python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01f_ncu1.out 2>&1
FAGP_GRAM_CFG=large timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -c 1 -o gpurun_out/r01f_gram_large python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r01f_ncu2.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r01f_ncu_launch.out 2>&1

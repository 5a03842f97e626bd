bash tools/gpu_check.sh r01o tests bench
FAGP_VAR_WARPS=4 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r01o_bench_w4.json 2>&1

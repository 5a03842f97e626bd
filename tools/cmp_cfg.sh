bash tools/gpu_check.sh r01g tests bench ncu
FAGP_PREDICT_CFG=large timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r01g_bench_plarge.json 2>&1

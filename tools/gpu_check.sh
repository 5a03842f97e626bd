#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the top kernels.
# Usage: bash tools/gpu_check.sh [tag] [stages...]   stages: tests smoke bench ncu full
set -u
TAG=${1:-r01}; shift || true
STAGES=${*:-"tests smoke bench ncu full"}
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc > gpurun_out/${TAG}_host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/${TAG}_host.txt
for s in $STAGES; do
  case $s in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt ;;
    testsall) timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt ;;
    sanitize) for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/${TAG}_san_${tool}.txt 2>&1; echo "$tool rc=$?" >> gpurun_out/${TAG}_san_${tool}.txt; done ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt ;;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err ;;
    benchref) timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.out 2>&1 ;;
    full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused_gram|fused_predict|cholinv_persistent|tiled_gram|tiled_predict" -c 3 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.out 2>&1 ;;
  esac
done
tail -3 gpurun_out/${TAG}_pytest_gpu.txt 2>/dev/null; cat gpurun_out/${TAG}_smoke.txt 2>/dev/null; cat gpurun_out/${TAG}_bench.json 2>/dev/null; tail -3 gpurun_out/${TAG}_bench.err 2>/dev/null

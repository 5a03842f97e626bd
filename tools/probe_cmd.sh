mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_probe > gpurun_out/fp64_probe.json 2>&1
python tools/dgemm_probe.py > gpurun_out/dgemm_probe.json 2>&1
kill $SMI
nvidia-smi -q | grep -i -E "Product Name|Max Clocks|Power Limit" | head > gpurun_out/smi.txt
cat gpurun_out/fp64_probe.json gpurun_out/dgemm_probe.json

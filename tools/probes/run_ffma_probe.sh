nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probes/ffma_probe > gpurun_out/ffma_probe.json 2>&1
kill $SMI
nproc > gpurun_out/host.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
cat gpurun_out/ffma_probe.json gpurun_out/host.txt

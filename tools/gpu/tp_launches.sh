# ncu launch list (time + DRAM bytes) of the TP bench step, summarised per kernel.
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"tp_|symcon_tp" --csv --log-file gpurun_out/tp_launches_${TAG:-x}.csv \
  python bench.py --channelwise-tp --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/tp_ncu_${TAG:-x}.log 2>&1; echo rc=$?
python tools/tp_launch_summary.py gpurun_out/tp_launches_${TAG:-x}.csv

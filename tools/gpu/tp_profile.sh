# TP round artifacts: bench line, launch list (time + DRAM bytes), one ncu --set full of the TP kernels.
export PYTHONUNBUFFERED=1
T=${TAG:-r01}
timeout 600 python bench.py --channelwise-tp --steps 10 --warmup 3 > gpurun_out/tp_bench_${T}.json 2> gpurun_out/tp_bench_${T}.err; echo bench_rc=$?
TAG=$T bash tools/gpu/tp_launches.sh > gpurun_out/tp_launch_summary_${T}.txt 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"symcon_tp_|tp_dh" -c 3 -o gpurun_out/prof_tp_${T} \
  python bench.py --channelwise-tp --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_tp_${T}.log 2>&1; echo full_rc=$?
tail -2 gpurun_out/ncu_tp_${T}.log

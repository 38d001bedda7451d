# Round profile: bench line, launch list of the same bench command, and one --set full capture.
export PYTHONUNBUFFERED=1
T=${TAG:-r01}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err; echo bench_rc=$?
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small_${T}.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"symcon|bk_|dw_" --csv \
  --log-file gpurun_out/launches_bench_${T}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_${T}.log 2>&1; echo launch_rc=$?
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain_${T}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"symcon_|bk_|dw_" -s 9 -c 9 -o gpurun_out/prof_full_${T} \
  python tools/profile_step.py > gpurun_out/ncu_full_${T}.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full_${T}.log

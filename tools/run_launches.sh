# Launch list (every kernel, device time) of one profile_step run, after a plain run exits 0.
export PYTHONUNBUFFERED=1
CFG=${CFG:-mp_medium}
timeout 300 python tools/profile_step.py --config $CFG > gpurun_out/launch_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-v}.csv \
  python tools/profile_step.py --config $CFG > gpurun_out/launch_ncu.log 2>&1
echo rc=$?

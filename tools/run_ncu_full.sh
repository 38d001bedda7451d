export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:symcon_ -s 6 -c 6 -o gpurun_out/prof_${TAG:-v} python tools/profile_step.py > gpurun_out/ncu_v1.log 2>&1
echo rc=$?
tail -5 gpurun_out/ncu_v1.log

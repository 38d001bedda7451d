export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_step.py --config large --iters 2 > gpurun_out/pl_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"symcon_bwd_dW|symcon_fwd" -s 2 -c 2 -o gpurun_out/prof_large python tools/profile_step.py --config large --iters 2 > gpurun_out/pl_ncu.log 2>&1; echo rc=$?

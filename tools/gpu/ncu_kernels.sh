# ncu --set full of selected kernels of tools/profile_step.py (one GPU).
#   CFG=large K="symcon_bwd_dW|symcon_bwd2_dW" S=3 C=2 TAG=x EXTRA=--bwd2 bash tools/gpu/ncu_kernels.sh
export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_step.py --config ${CFG:-mp_medium} --iters 2 $EXTRA > gpurun_out/pk_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s ${S:-0} -c ${C:-2} -o gpurun_out/prof_${TAG:-k} python tools/profile_step.py --config ${CFG:-mp_medium} --iters 2 $EXTRA > gpurun_out/pk_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/pk_ncu.log

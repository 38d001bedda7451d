# ncu --set full of the R kernels (fwd_r, dW_r) on the MP-medium shape
V="$1"
python tools/variants.py --config mp_medium --iters 3 "$V" > gpurun_out/plain_r.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"symcon_fwd_r|symcon_bwd_dW_r|symcon_bwd_dA" -s 6 -c 3 -o gpurun_out/prof_r python tools/variants.py --config mp_medium --iters 3 "$V" > gpurun_out/ncu_r.log 2>&1
tail -3 gpurun_out/ncu_r.log

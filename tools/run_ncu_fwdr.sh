python tools/variants.py --config mp_medium --iters 3 "fwd_r=1,fwd_r_block=16" > gpurun_out/plain_fwdr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:symcon_fwd_r -s 2 -c 1 -o gpurun_out/prof_fwdr python tools/variants.py --config mp_medium --iters 3 "fwd_r=1,fwd_r_block=16" > gpurun_out/ncu_fwdr.log 2>&1
tail -3 gpurun_out/ncu_fwdr.log

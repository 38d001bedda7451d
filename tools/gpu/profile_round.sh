# Round-2 profile set (profiles/r02): bench line (N = 1 defaults), the ncu launch list of the same bench
# command, and one ncu --set full capture (+ FP32 op counters, local-memory bytes) of every kernel of a
# tools/profile_step.py fwd+bwd step on MP-medium (50k nodes).
export PYTHONUNBUFFERED=1
T=${TAG:-r02}
OPS=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_data_bytes_mem_local_op_ld.sum,sm__sass_data_bytes_mem_local_op_st.sum
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err; echo bench_rc=$?
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small_${T}.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"symcon|bk_|dw_" --csv \
  --log-file gpurun_out/launches_bench_${T}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_${T}.log 2>&1; echo launch_rc=$?
timeout 300 python tools/profile_step.py --iters 2 > gpurun_out/prof_plain_${T}.log 2>&1 && \
timeout 1200 ncu --set full --metrics $OPS --clock-control none --import-source on -k regex:"symcon_|bk_|dw_" -c 16 -o gpurun_out/prof_full_${T} \
  python tools/profile_step.py --iters 2 > gpurun_out/ncu_full_${T}.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full_${T}.log

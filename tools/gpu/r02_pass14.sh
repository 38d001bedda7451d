# Round-2 pass 14: dW_r CTAs of single-item elements unfold dW themselves (dw_r_unfold_single).
export PYTHONUNBUFFERED=1
D=gpurun_out/r02p; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_step.py -x -q > $D/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest.log
BENCH_ARGS="--capacity 3072" bash tools/gpu/kconfig_sweep.sh "" "dw_r_unfold_single=0" > $D/sweep_c3072.jsonl 2>&1; cat $D/sweep_c3072.jsonl
bash tools/gpu/kconfig_sweep.sh "" "dw_r_unfold_single=0" > $D/sweep_50k.jsonl 2>&1; cat $D/sweep_50k.jsonl
BENCH_ARGS="--config off_small" bash tools/gpu/kconfig_sweep.sh "" "dw_r_unfold_single=0" > $D/sweep_off.jsonl 2>&1; cat $D/sweep_off.jsonl

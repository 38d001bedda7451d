# Round-2 pass 8: OFF-small dW_r with several warps per slot (dw_r_wps): parity on the OFF shapes, then A/B.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02i; mkdir -p $D
SYMCON_KCONFIG="dw_r=1" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $D/pytest_dwr_wps.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_dwr_wps.log
BENCH_ARGS="--config off_small" bash tools/gpu/kconfig_sweep.sh "" "dw_r=1,dw_r_wps=1" "dw_r=1,dw_r_wps=2" "dw_r=1,dw_r_wps=4" "dw_r=1,dw_r_wps=8" "dw_r=1,dw_r_wps=4,dw_r_block=16" > $D/sweep_off_dw.jsonl 2>&1
cat $D/sweep_off_dw.jsonl

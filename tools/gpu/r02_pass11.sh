# Round-2 pass 11: dW_r with row-group sets (grid.z) on the 9-slot large shape: parity, then A/B.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02m; mkdir -p $D
SYMCON_KCONFIG="dw_r=1" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not backward2 and not double" > $D/pytest_dwr_large.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_dwr_large.log
BENCH_ARGS="--config large --steps 6 --warmup 3" bash tools/gpu/kconfig_sweep.sh "" "dw_r=1" "dw_r=1,dw_r_minb=2" > $D/sweep_large_dw.jsonl 2>&1
cat $D/sweep_large_dw.jsonl

# Round-2 pass 10: fwd_r with slot groups on the 9-slot large shape: parity, then A/B.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02l; mkdir -p $D
SYMCON_KCONFIG="fwd_r=1" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not backward2 and not double" > $D/pytest_fwdr_large.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_fwdr_large.log
BENCH_ARGS="--config large --steps 6 --warmup 3" bash tools/gpu/kconfig_sweep.sh "" "fwd_r=1" "fwd_r=1,fwd_r_minb=4" "fwd_r=1,fwd_r_minb=5" "fwd_r=1,fwd_r_minb=2" > $D/sweep_large.jsonl 2>&1
cat $D/sweep_large.jsonl

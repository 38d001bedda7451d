# Round-2 pass 9: full GPU suite with dW_r on one-slot plans and the gamma dA tile split; OFF A/B of the split.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02j; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_gpu.log
BENCH_ARGS="--config off_small" bash tools/gpu/kconfig_sweep.sh "" "gamma_split=1" "gamma_split=2" "gamma_split=3" "gamma_split=4" > $D/sweep_off_gs.jsonl 2>&1
cat $D/sweep_off_gs.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $D/bench_n1.json 2> $D/bench_n1.err; echo n1_rc=$?
head -c 300 $D/bench_n1.json

# Round-2 pass 13: single-item elements' dW rows written straight into the reduced table.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02o; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_step.py -x -q > $D/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest.log
timeout 600 python bench.py --capacity 3072 --steps 50 --warmup 5 --no-cpu-baseline > $D/bench_c3072.json 2> $D/bench_c3072.err; echo c_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $D/bench_n1.json 2> $D/bench_n1.err; echo n1_rc=$?
timeout 600 python bench.py --config off_small --steps 20 --warmup 5 --no-cpu-baseline > $D/bench_off.json 2> $D/bench_off.err; echo off_rc=$?
for f in $D/*.json; do echo $f; head -c 230 $f; echo; done

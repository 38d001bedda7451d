# Round-2 GPU pass 4: simple-plan dW with CTA-shared node staging (fp64 / corr 4), full-size variant
# parity, fp64 / corr-4 bench lines, C = 3072 with and without the small-N dW item size.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02d; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_f64.py tests/test_gpu_corr4.py tests/test_gpu_timed_step.py -x -q > $D/pytest_variants.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_variants.log
timeout 600 python bench.py --steps 10 --warmup 3 --dtype f64 --cpu-sample 8192 > $D/bench_f64.json 2> $D/bench_f64.err; echo f64_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --correlation 4 --cpu-sample 1024 > $D/bench_corr4.json 2> $D/bench_corr4.err; echo c4_rc=$?
SYMCON_KCONFIG=dw_items_adapt=0 timeout 600 python bench.py --steps 50 --warmup 5 --capacity 3072 --no-cpu-baseline > $D/bench_c3072_noadapt.json 2> $D/bench_c3072_noadapt.err; echo na_rc=$?
timeout 600 python bench.py --steps 50 --warmup 5 --capacity 3072 > $D/bench_c3072.json 2> $D/bench_c3072.err; echo c3072_rc=$?
for f in $D/*.json; do echo $f; head -c 200 $f; echo; done

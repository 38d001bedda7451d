# Round-2 GPU pass 3: GPU tests after the fold/bucket fork and the small-N dW item size; bench lines at
# C = 50k and C = 3072 with the fork on / off; fp64 line after the dW prefix sharing.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02c; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench_n1.json 2> $D/bench_n1.err; echo n1_rc=$?
SYMCON_KCONFIG=fold_fork=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $D/bench_n1_nofork.json 2> $D/bench_n1_nofork.err; echo n1nf_rc=$?
timeout 600 python bench.py --steps 50 --warmup 5 --capacity 3072 --no-cpu-baseline > $D/bench_c3072.json 2> $D/bench_c3072.err; echo c3072_rc=$?
SYMCON_KCONFIG=fold_fork=0 timeout 600 python bench.py --steps 50 --warmup 5 --capacity 3072 --no-cpu-baseline > $D/bench_c3072_nofork.json 2> $D/bench_c3072_nofork.err; echo c3072nf_rc=$?
SYMCON_KCONFIG=dw_tiles_per_item=4,fold_fork=1 timeout 600 python bench.py --steps 50 --warmup 5 --capacity 3072 --no-cpu-baseline > $D/bench_c3072_tpi4.json 2> $D/bench_c3072_tpi4.err; echo c3072t_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --dtype f64 --no-cpu-baseline > $D/bench_f64.json 2> $D/bench_f64.err; echo f64_rc=$?
for f in $D/*.json; do echo $f; head -c 200 $f; echo; done

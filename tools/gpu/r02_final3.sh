# Round-2 closing 1-GPU pass on the final code: smoke, full GPU suite, the profile set, every N = 1 line.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02y; mkdir -p $D
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_gpu.log
TAG=r02y bash tools/gpu/profile_round.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_reference.json 2> $D/bench_reference.err; echo ref_rc=$?
timeout 600 python bench.py --config off_small --steps 20 --warmup 5 > $D/bench_off_small.json 2> $D/bench_off_small.err; echo off_rc=$?
timeout 900 python bench.py --config large --steps 10 --warmup 3 --cpu-sample 2048 > $D/bench_large.json 2> $D/bench_large.err; echo large_rc=$?
timeout 600 python bench.py --capacity 3072 --steps 50 --warmup 5 > $D/bench_c3072.json 2> $D/bench_c3072.err; echo c3072_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --dtype f64 --cpu-sample 8192 > $D/bench_f64.json 2> $D/bench_f64.err; echo f64_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --correlation 4 --cpu-sample 1024 > $D/bench_corr4.json 2> $D/bench_corr4.err; echo c4_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --double-backward --no-cpu-baseline > $D/bench_dbl.json 2> $D/bench_dbl.err; echo dbl_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --channelwise-tp --no-cpu-baseline > $D/bench_tp.json 2> $D/bench_tp.err; echo tp_rc=$?
for f in $D/*.json gpurun_out/bench_r02y.json; do echo $f; head -c 200 $f; echo; done

# Round-2 final N = 1 variant lines on the final code: fp64, correlation 4, force-training step, headline.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02h; mkdir -p $D
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench_n1.json 2> $D/bench_n1.err; echo n1_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --dtype f64 --cpu-sample 8192 > $D/bench_f64.json 2> $D/bench_f64.err; echo f64_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --correlation 4 --cpu-sample 1024 > $D/bench_corr4.json 2> $D/bench_corr4.err; echo c4_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --double-backward --no-cpu-baseline > $D/bench_dbl.json 2> $D/bench_dbl.err; echo dbl_rc=$?
for f in $D/*.json; do echo $f; head -c 200 $f; echo; done

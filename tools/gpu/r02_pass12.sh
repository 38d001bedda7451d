# Round-2 pass 12: full GPU suite on the final defaults, large and MP lines.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02n; mkdir -p $D
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_gpu.log
timeout 900 python bench.py --config large --steps 10 --warmup 3 --cpu-sample 2048 > $D/bench_large.json 2> $D/bench_large.err; echo large_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench_n1.json 2> $D/bench_n1.err; echo n1_rc=$?
for f in $D/*.json; do echo $f; head -c 250 $f; echo; done

# Round-2 pass 7: C = 3072 with the L2 flush (N = 1), small-N tail options A/B at C = 3072.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02g; mkdir -p $D
timeout 600 python bench.py --capacity 3072 --steps 50 --warmup 5 > $D/bench_c3072.json 2> $D/bench_c3072.err; echo c3072_rc=$?
BENCH_ARGS="--capacity 3072" bash tools/gpu/kconfig_sweep.sh "" "unfold_reduce=1" "bucket_fused=1" "unfold_reduce=1,bucket_fused=1" "fold_fork=0" > $D/sweep_c3072.jsonl 2>&1
cat $D/sweep_c3072.jsonl
head -c 400 $D/bench_c3072.json

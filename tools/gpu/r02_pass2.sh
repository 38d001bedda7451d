# Round-2 GPU pass 2: full GPU test suite, the FP64 DFMA probe, fp64 / correlation-4 bench lines,
# the double-backward register-cap comparison (bwd2_min_blocks 10 vs 8), TP bench with graph reuse.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r02b/pytest_gpu.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/dfma_probe tools/probes/dfma_probe.cu && \
  timeout 120 tools/probes/dfma_probe > gpurun_out/r02b/dfma_probe.jsonl 2>&1; echo dfma_rc=$?
mkdir -p profiles/r02 && cp gpurun_out/r02b/dfma_probe.jsonl profiles/r02/dfma_probe.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 --dtype f64 --cpu-sample 8192 > gpurun_out/r02b/bench_f64.json 2> gpurun_out/r02b/bench_f64.err; echo f64_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --correlation 4 --cpu-sample 1024 > gpurun_out/r02b/bench_corr4.json 2> gpurun_out/r02b/bench_corr4.err; echo c4_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --double-backward --no-cpu-baseline > gpurun_out/r02b/bench_dbl_minb10.json 2> gpurun_out/r02b/bench_dbl_minb10.err; echo dbl10_rc=$?
SYMCON_KCONFIG=bwd2_min_blocks=8 timeout 900 python bench.py --steps 20 --warmup 5 --double-backward --no-cpu-baseline > gpurun_out/r02b/bench_dbl_minb8.json 2> gpurun_out/r02b/bench_dbl_minb8.err; echo dbl8_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --channelwise-tp --no-cpu-baseline > gpurun_out/r02b/bench_tp.json 2> gpurun_out/r02b/bench_tp.err; echo tp_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b/bench_n1.json 2> gpurun_out/r02b/bench_n1.err; echo n1_rc=$?
for f in gpurun_out/r02b/*.json; do echo $f; head -c 250 $f; echo; done

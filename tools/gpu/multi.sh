# N-GPU runs (gpurun --gpus N): multi-GPU tests, bench lines for the one-shot / two-shot peer all-reduce and NCCL,
# at C = 50,000 and at the paper's C = 3072 (CUDA-graph replay of the whole step, --graph-all)
N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
mkdir -p gpurun_out/multi_n$N
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_n$N/pytest_multi.log 2>&1
for algo in 1 2; do
  timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --peer-algo $algo > gpurun_out/multi_n$N/bench_c50k_algo$algo.json 2> gpurun_out/multi_n$N/bench_c50k_algo$algo.err
  timeout 300 $TR bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline --peer-algo $algo --capacity 3072 --graph-all > gpurun_out/multi_n$N/bench_c3072_algo$algo.json 2> gpurun_out/multi_n$N/bench_c3072_algo$algo.err
done
timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --allreduce nccl > gpurun_out/multi_n$N/bench_c50k_nccl.json 2> gpurun_out/multi_n$N/bench_c50k_nccl.err
timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --graph-all > gpurun_out/multi_n$N/bench_c50k_graph.json 2> gpurun_out/multi_n$N/bench_c50k_graph.err
tail -3 gpurun_out/multi_n$N/pytest_multi.log
for f in gpurun_out/multi_n$N/*.json; do echo $f; head -c 300 $f; echo; done

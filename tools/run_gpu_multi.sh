# Multi-GPU bench on one box: N=1 then N=$NG via torchrun (NCCL), same workload per GPU.
export PYTHONUNBUFFERED=1
NG=${NG:-2}
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo n1_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo n${NG}_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --no-overlap > gpurun_out/bench_n${NG}_noov.json 2> gpurun_out/bench_n${NG}_noov.err; echo n${NG}_noov_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
for f in gpurun_out/bench_n1.json gpurun_out/bench_n$NG.json gpurun_out/bench_n${NG}_noov.json gpurun_out/bench_ref.json; do python -c "
import json,sys
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1])
  print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), d.get('per_gpu_nodes_per_s'), d.get('config',{}).get('step_imbalance_max_over_mean'))
except Exception as e: print('$f', 'ERR', e)
"; done
tail -5 gpurun_out/bench_n$NG.err

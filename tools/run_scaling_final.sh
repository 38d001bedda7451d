# Final scaling set: N=1,2,4 default bench lines (+ N=4 with NCCL), JSON in gpurun_out/sf_*.json.
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/sf_n1.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/sf_n2.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --steps 50 --warmup 5 > gpurun_out/sf_n4.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29673 bench.py --gpus 4 --steps 50 --warmup 5 --allreduce nccl --no-cpu-baseline > gpurun_out/sf_n4_nccl.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29674 bench.py --gpus 4 --steps 20 --warmup 5 --double-backward --no-cpu-baseline > gpurun_out/sf_n4_dbl.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29675 bench.py --gpus 4 --steps 10 --warmup 3 --channelwise-tp --no-cpu-baseline > gpurun_out/sf_n4_tp.json 2>/dev/null
for f in n1 n2 n4 n4_nccl n4_dbl n4_tp; do python -c "
import json
d=json.loads(open('gpurun_out/sf_$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['value']/1e6,2), round(d['ms_per_step'],3), d.get('per_rank_ms_per_step'), d['clocks']['samples'])"; done

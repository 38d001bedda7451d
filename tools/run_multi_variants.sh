# N-GPU variants of the data-parallel step (overlap/concurrency/NCCL channel settings)
export PYTHONUNBUFFERED=1
NG=${NG:-2}
run() { tag=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
  bench.py --gpus $NG --steps 20 --warmup 5 --no-cpu-baseline $EXTRA > gpurun_out/mv_$tag.json 2> gpurun_out/mv_$tag.err;
  python -c "
import json
d=json.loads(open('gpurun_out/mv_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['per_gpu_nodes_per_s']/1e6,2))" ; }
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mv_n1.json 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/mv_n1.json').read().strip().splitlines()[-1]); print('n1', round(d['value']/1e6,2), round(d['ms_per_step'],4))"
EXTRA="" run conc
EXTRA="--sequential-bwd" run seq
EXTRA="" run conc_ch2 NCCL_MAX_NCHANNELS=2
EXTRA="--sequential-bwd" run seq_ch2 NCCL_MAX_NCHANNELS=2
EXTRA="" run conc_nvls NCCL_NVLS_ENABLE=1 NCCL_MAX_NCHANNELS=4

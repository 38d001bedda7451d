# Scaling table: N=1 and N=$NG for the default DP step (repeated), JSON lines in gpurun_out/scal_<tag>_*.json.
export PYTHONUNBUFFERED=1
NG=${NG:-4}
T=${TAG:-x}
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scal_${T}_n1.json 2>/dev/null
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2957$rep \
  bench.py --gpus $NG --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scal_${T}_n${NG}_$rep.json 2>/dev/null
done
for f in gpurun_out/scal_${T}_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['value']/1e6,2), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; done

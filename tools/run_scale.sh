# Scaling on one box: N=1 and N=$NG (torchrun, NCCL) for the default step and the
# force-training step (--double-backward); JSON lines in gpurun_out/scale_<tag>_*.json.
export PYTHONUNBUFFERED=1
NG=${NG:-4}
T=${TAG:-s}
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_${T}_n1.json 2> gpurun_out/scale_${T}_n1.err; echo n1_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus $NG --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_${T}_n$NG.json 2> gpurun_out/scale_${T}_n$NG.err; echo n${NG}_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --double-backward > gpurun_out/scale_${T}_n1_dbl.json 2> gpurun_out/scale_${T}_n1_dbl.err; echo n1dbl_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29519 \
  bench.py --gpus $NG --steps 10 --warmup 3 --no-cpu-baseline --double-backward > gpurun_out/scale_${T}_n${NG}_dbl.json 2> gpurun_out/scale_${T}_n${NG}_dbl.err; echo n${NG}dbl_rc=$?
for f in gpurun_out/scale_${T}_*.json; do python -c "
import json
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1])
  print('$f', d.get('metric'), d.get('n_gpus'), round(d.get('value')/1e6, 2), round(d.get('ms_per_step'), 3), d.get('clocks',{}).get('sm_mhz'))
except Exception as e: print('$f', 'ERR', e)
"; done
tail -3 gpurun_out/scale_${T}_n$NG.err

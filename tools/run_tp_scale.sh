# TP weak scaling (no data-path collective) and the contraction DP step at N=$NG.
export PYTHONUNBUFFERED=1
NG=${NG:-4}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -9 gpurun_out/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29521 \
  bench.py --gpus $NG --channelwise-tp --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tp_scale_n$NG.json 2> gpurun_out/tp_scale_n$NG.err; echo tp_n${NG}_rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/tp_scale_n$NG.json').read().strip().splitlines()[-1]); print('tp', d['n_gpus'], round(d['value']/1e6,1), round(d['ms_per_step'],3))"

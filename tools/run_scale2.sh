# N=$NG runs of the three bench modes (default DP step, force-training step, channelwise TP).
export PYTHONUNBUFFERED=1
NG=${NG:-2}
T=${TAG:-s2}
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $1 \
  bench.py --gpus $NG --steps 20 --warmup 5 --no-cpu-baseline $2 > gpurun_out/${T}_$3.json 2> gpurun_out/${T}_$3.err; echo $3 rc=$?; }
run 29531 "" dp
run 29532 "--double-backward" dbl
run 29533 "--channelwise-tp" tp
for f in dp dbl tp; do python -c "
import json
d=json.loads(open('gpurun_out/${T}_$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['value']/1e6,2), round(d['ms_per_step'],3), d['clocks']['samples'])"; done

export PYTHONUNBUFFERED=1
for c in off_small large; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-sample 1024 > gpurun_out/bench_cfg_$c.json 2> gpurun_out/bench_cfg_$c.err; echo $c rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['path_frac_of_alu_peak'],3), d['kernels'], d['cpu_baseline']['value'])"
done
tail -3 gpurun_out/bench_cfg_large.err

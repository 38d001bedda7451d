export PYTHONUNBUFFERED=1
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_seq$i.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --concurrent-bwd > gpurun_out/bench_cc$i.json 2>&1
done
for f in gpurun_out/bench_seq1.json gpurun_out/bench_cc1.json gpurun_out/bench_seq2.json gpurun_out/bench_cc2.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), round(d['ms_per_step'],4))"; done

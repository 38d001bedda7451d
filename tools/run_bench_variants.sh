# bench.py (N=1, default concurrent dW || dA) under several SYMCON_KCONFIG variants.
#   VARS="base da_ctas_per_sm=8,dw_groups_per_cta=4" TAG=x bash tools/run_bench_variants.sh
export PYTHONUNBUFFERED=1
for v in $VARS; do
  if [ "$v" = "base" ]; then export SYMCON_KCONFIG=""; else export SYMCON_KCONFIG="$v"; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $EXTRA > gpurun_out/bv_${TAG}_tmp.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bv_${TAG}_tmp.json').read().strip().splitlines()[-1])
print(json.dumps({'variant': '$v', 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'kernels': {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()}, 'clocks': d['clocks']['sm_mhz']}))
" >> gpurun_out/bv_${TAG}.jsonl
done
cat gpurun_out/bv_${TAG}.jsonl

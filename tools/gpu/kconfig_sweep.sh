# bench.py (N=1, default workload + $BENCH_ARGS) under several SYMCON_KCONFIG variants; one JSON line each
for v in "$@"; do
  SYMCON_KCONFIG="$v" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $BENCH_ARGS > gpurun_out/bkc.json 2> gpurun_out/bkc.err
  python - "$v" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bkc.json"))
    print(json.dumps({"kconfig": sys.argv[1], "value": d["value"], "ms_per_step": d["ms_per_step"],
                      "path_frac": d["path_roofline"]["frac"], "kernels": {k: round(x["avg_ms"], 4) for k, x in d["kernels"].items()}}))
except Exception as e:
    print(json.dumps({"kconfig": sys.argv[1], "error": str(e), "stderr": open("gpurun_out/bkc.err").read()[-500:]}))
PY
done

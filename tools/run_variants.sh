export PYTHONUNBUFFERED=1
V=${V:-""}
timeout 1500 python tools/variants.py $V > gpurun_out/variants_${TAG:-x}.jsonl 2> gpurun_out/variants_${TAG:-x}.err; echo rc=$?
cat gpurun_out/variants_${TAG:-x}.jsonl | cut -c1-330; tail -3 gpurun_out/variants_${TAG:-x}.err

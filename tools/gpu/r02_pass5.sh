# Round-2 GPU pass 5: fwd_r with two warps per output slot (fwd_r_split=2) -- parity, then A/B lines.
export PYTHONUNBUFFERED=1
D=gpurun_out/r02e; mkdir -p $D
SYMCON_KCONFIG="fwd_r_split=2,fwd_r_minb=2" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $D/pytest_parity_split.log 2>&1; echo pytest_rc=$?; tail -2 $D/pytest_parity_split.log
bash tools/gpu/kconfig_sweep.sh "" "fwd_r_chains=2" "fwd_r_split=2,fwd_r_minb=2" "fwd_r_split=2,fwd_r_minb=2,fwd_r_chains=2" "fwd_r_split=2,fwd_r_minb=0" > $D/sweep.jsonl 2>&1
cat $D/sweep.jsonl

"""Compile a plan's generated kernels here (no GPU) and print registers / spills per kernel.

    python tools/regcheck.py [--config mp_medium] "" "dw_rows_per_group=64,dw_groups_per_cta=8" ...
"""
import argparse
import ctypes
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mp_medium")
    ap.add_argument("variants", nargs="*", default=[""])
    args = ap.parse_args()
    from paper_2504_10700_b200 import _lib
    from synth.inputs import CONFIGS
    cfg = CONFIGS[args.config]
    out_dir = os.path.join(ROOT, "gpurun_out", "src")
    os.makedirs(out_dir, exist_ok=True)
    for v in args.variants:
        os.environ["SYMCON_KCONFIG"] = v
        plan = _lib.symcon_build_tables(cfg.lmax_in, cfg.correlation, list(cfg.out_L), cfg.n_elements, cfg.channels, -1)
        n = _lib.lib.symcon_plan_source(plan, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        _lib.lib.symcon_plan_source(plan, buf, n + 1)
        _lib.symcon_destroy(plan)
        src = os.path.join(out_dir, "regcheck.cu")
        open(src, "wb").write(buf.value)
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-std=c++17", "-Xptxas", "-v",
                            "-o", os.path.join(out_dir, "regcheck.cubin"), src], capture_output=True, text=True)
        res = {}
        cur = None
        for line in r.stderr.splitlines():
            m = re.search(r"Compiling entry function '(\w+)'", line)
            if m:
                cur = m.group(1)
            m = re.search(r"(\d+) bytes spill stores", line)
            if m and cur:
                res.setdefault(cur, {})["spill"] = int(m.group(1))
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                res.setdefault(cur, {})["regs"] = int(m.group(1))
        print(repr(v), " ".join(f"{k}:{d.get('regs')}/{d.get('spill')}" for k, d in sorted(res.items())), flush=True)


if __name__ == "__main__":
    main()

"""Instruction mix of the generated kernels of one configuration (CPU-only: NVRTC + cuobjdump).

    python tools/sass_mix.py 3 3 0,1
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    lmax, corr = int(sys.argv[1]), int(sys.argv[2])
    outs = [int(x) for x in sys.argv[3].split(",")]
    from paper_2504_10700_b200 import build_lib
    build_lib.build()
    from paper_2504_10700_b200 import _lib
    path = _lib.symcon_precompile(lmax, corr, outs)
    log = open(path.replace(".cubin", ".log"), errors="replace").read()
    for m in re.finditer(r"Compiling entry function '(\w+)'.*?\n.*?(\d+) bytes spill stores.*?\n.*?Used (\d+) registers", log, re.S):
        print(f"{m.group(1):16s} regs={m.group(3)} spill_st={m.group(2)}")
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn = None
    mix = collections.defaultdict(collections.Counter)
    for line in sass.splitlines():
        m = re.search(r"Function : (\w+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?P\d\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            mix[fn][m.group(2)] += 1
    for f, c in mix.items():
        tot = sum(c.values())
        print(f, tot, dict(c.most_common(10)))


if __name__ == "__main__":
    main()

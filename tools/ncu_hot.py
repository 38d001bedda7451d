"""Top stalled SASS instructions of one kernel in an ncu report.

    python tools/ncu_hot.py gpurun_out/prof_v3.ncu-rep symcon_fwd [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, n=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    data = rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[si] or 0) for r in data)
    agg = {c: sum(int(r[hdr.index(c)] or 0) for r in data) for c in cols}
    print("samples", tot, sorted(((k, round(v / tot, 3)) for k, v in agg.items()), key=lambda x: -x[1])[:8])
    for i, r in enumerate(sorted(range(len(data)), key=lambda i: -int(data[i][si] or 0))[:n]):
        row = data[r]
        st = {c: int(row[hdr.index(c)] or 0) for c in cols}
        st = sorted(((k, v) for k, v in st.items() if v), key=lambda x: -x[1])[:3]
        print(f"{row[si]:>6} #{r:5d} {row[src].strip()[:64]:64s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)

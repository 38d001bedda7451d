"""Per-kernel summary (last occurrence) of an ncu --csv launch list with time and DRAM bytes."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = {}
for r in data:
    per.setdefault(r[ii], {"k": r[ki].split("(")[0].replace("symcon::<unnamed>::", "")})[r[mi]] = float(r[vi].replace(",", ""))
last = {}
for i in sorted(per, key=int):
    last[per[i]["k"]] = per[i]
for k, m in last.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd, wr = m.get("dram__bytes_read.sum", 0) / 1e9, m.get("dram__bytes_write.sum", 0) / 1e9
    print(f"{k:24s} {t:9.1f} us  read {rd:7.3f} GB  write {wr:7.3f} GB  {((rd + wr) / (t / 1e6) if t else 0):7.0f} GB/s")

"""Write profiles/<round>/ artifacts from a tools/gpu/profile_round.sh capture.

    python tools/make_profile_artifacts.py r01c profiles/r01
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_list(tag, out_dir):
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"launches_bench_{tag}.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    seq = [(r[ii], r[ki].split("(")[0], float(r[vi].replace(",", ""))) for r in data if r[mi] == "gpu__time_duration.sum"]
    tot = {}
    for _, k, v in seq:
        tot[k] = tot.get(k, 0) + v
    s = sum(tot.values())
    with open(os.path.join(out_dir, "launch_list_bench.txt"), "w") as f:
        f.write(f"# capture {tag}: ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'symcon|bk_|dw_' "
                "python bench.py --steps 2 --warmup 1 --no-cpu-baseline\n")
        f.write("# per-launch device time (cold-cache, serialised by ncu); per-kernel share of the summed time\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{k:40s} total {v / 1000:9.1f} us  share {100 * v / s:5.1f}%\n")
        f.write("\n# launches\n")
        for i, k, v in seq:
            f.write(f"{i:>5} {k:40s} {v / 1000:9.1f} us\n")


def traffic(tag, out_dir):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_full_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        if name in out:
            continue

        def v(k, table):
            return float(d[k].replace(",", "")) * table.get(units[hdr.index(k)], 1)
        rec = {"dram_bytes_read": v("dram__bytes_read.sum", scale), "dram_bytes_write": v("dram__bytes_write.sum", scale),
               "time_us": v("gpu__time_duration.sum", tscale),
               "fma_pipe_pct": float(d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]),
               "issue_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
               "registers": int(float(d["launch__registers_per_thread"]))}
        # executed FP32 lane-ops (thread instructions; the packed forms do 2 lane-ops each) and local bytes
        ops = {k: d.get(f"sm__sass_thread_inst_executed_op_{k}_pred_on.sum") for k in ("ffma", "ffma2", "fmul", "fmul2", "fadd", "fadd2")}
        if all(x not in (None, "") for x in ops.values()):
            ops = {k: float(x.replace(",", "")) for k, x in ops.items()}
            rec["thread_inst"] = ops
            rec["executed_lane_ops"] = ops["ffma"] + ops["fmul"] + ops["fadd"] + 2 * (ops["ffma2"] + ops["fmul2"] + ops["fadd2"])
        for k, key in (("local_ld_bytes", "sm__sass_data_bytes_mem_local_op_ld.sum"), ("local_st_bytes", "sm__sass_data_bytes_mem_local_op_st.sum")):
            if d.get(key) not in (None, ""):
                rec[k] = v(key, scale)
        out[name] = rec
        # the bench reports kernels by launch group (symcon_fwd covers symcon_fwd_r, ...)
        alias = {"symcon_fwd_r": "symcon_fwd", "symcon_bwd_dW_r": "symcon_bwd_dW", "symcon_bwd_dA_s": "symcon_bwd_dA"}.get(name)
        if alias and alias not in out:
            out[alias] = dict(rec, kernel=name)
    json.dump({"source": f"ncu --set full --clock-control none, tools/profile_step.py (MP-medium, 50k nodes), capture {tag}",
               "kernels": out}, open(os.path.join(out_dir, "ncu_traffic.json"), "w"), indent=1)
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True, text=True).stdout
    open(os.path.join(out_dir, "ncu_full_summary.txt"), "w").write(f"# capture {tag}\n" + summ)


if __name__ == "__main__":
    tag, out_dir = sys.argv[1], sys.argv[2]
    os.makedirs(out_dir, exist_ok=True)
    launch_list(tag, out_dir)
    traffic(tag, out_dir)
    import shutil
    shutil.copy(os.path.join(ROOT, "gpurun_out", f"bench_{tag}.json"), os.path.join(out_dir, f"bench_n1_{tag}.json"))
    print(open(os.path.join(out_dir, "launch_list_bench.txt")).read()[:900])

"""Summarise an ncu report (per kernel: time, pipe utilisation, DRAM bytes, occupancy, top stalls).

    python tools/ncu_summary.py gpurun_out/prof_v2.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time_us",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe%",
    "sm__inst_executed_pipe_fma.sum": "fma_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "launch__registers_per_thread": "regs",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "smsp__inst_executed.sum": "inst",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_conf",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum": "local_ld",
    "launch__grid_size": "grid",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma",
    "sm__sass_thread_inst_executed_op_ffma2_pred_on.sum": "ffma2",
    "sm__sass_thread_inst_executed_op_fmul_pred_on.sum": "fmul",
    "sm__sass_thread_inst_executed_op_fmul2_pred_on.sum": "fmul2",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum": "fadd",
    "sm__sass_data_bytes_mem_local_op_ld.sum": "local_ld_B",
    "sm__sass_data_bytes_mem_local_op_st.sum": "local_st_B",
}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out = {v: d.get(k) for k, v in KEYS.items()}
        unit = {v: units[hdr.index(k)] if k in hdr else "" for k, v in KEYS.items()}
        stalls = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v or 0))
                  for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -x[1])[:6]
        print(d["Kernel Name"], " ".join(f"{k}={v}{unit[k] if k.startswith('dram') or k == 'time_us' else ''}" for k, v in out.items()))
        print("   stalls:", ", ".join(f"{k}={v:.2f}" for k, v in stalls))


if __name__ == "__main__":
    main(sys.argv[1])

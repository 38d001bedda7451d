"""Benchmark: symmetric-contraction fwd+bwd nodes/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config mp_medium]
                    [--capacity C]

A step is one pass of the whole hot path over one bin of molecular graphs per GPU:
element bucketing, W-fold, forward B, backward dW (S partials + fixed-order reduction) and
dA, and -- for N > 1 -- the dW all-reduce (libsymcon's NVLink peer-memory kernel). Workload
(SURVEY.md §8(d) config 5 at the MP-medium shape): the 2,650,823-graph Table-2 manifest packed
by Alg. 1 (C++ partitioner, capacity C = 50,000 nodes by default, 3,072 = the paper's operating
point PAPER.md:969 with --capacity 3072, M = multiple of N bins), bin s*N + r on rank r at step s;
128 channels, 0e+1o output, lmax 3, correlation 3, 89 elements (1-4 Zipf elements per graph).
Inputs for the timed steps are resident in HBM before timing; A alone is 410 MB per 50k-node bin,
larger than L2, and a pool of distinct bins is cycled (at C = 3072 the 4-bin pool is L2-resident;
the line says so).

The exact timed step is `TimedStep` (also driven by tests/test_gpu_timed_step.py, which checks
its outputs against the oracle). One JSON line on rank 0. `roofline` reports the dominant
kernel, its per-launch CUDA-event time measured by libsymcon's launch timer.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CAPACITY = 50_000
# BASELINE.json configs: MP-medium = a 50k-node batch, large = a 200k-node batch (both Alg. 1 bins of the
# Table-2 manifest), OFF-small = a 20k-node batch of 10-100-atom molecules (organic element mix)
DEFAULT_CAPACITY = {"mp_medium": 50_000, "large": 200_000, "off_small": None}
OFF_BATCH_NODES = 20_000
POOL = 4
L2_BYTES = 126e6   # B200 L2
EDGE_DEGREE = 30   # synthetic in-degree min(30, n-1)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mp_medium", choices=["off_small", "mp_medium", "large"])
    ap.add_argument("--capacity", type=int, default=None,
                    help="Alg. 1 bin capacity in nodes per GPU-step (default: 50,000 mp_medium, 200,000 large; "
                         "the paper's 3072, PAPER.md:969); off_small uses 20k-node molecule batches instead")
    ap.add_argument("--cpu-sample", type=int, default=32768, help="nodes in the oracle's bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="all-reduce dW after dA instead of overlapping")
    ap.add_argument("--allreduce", default="peer", choices=["peer", "nccl"],
                    help="N > 1: dW all-reduce by libsymcon's NVLink peer-memory kernel (default) or NCCL")
    ap.add_argument("--peer-algo", type=int, default=0, choices=[0, 1, 2],
                    help="peer all-reduce: 0 auto (two-shot at N >= 8), 1 one-shot, 2 two-shot")
    ap.add_argument("--sequential-bwd", action="store_true", help="run the dW and dA kernels back to back on one stream")
    ap.add_argument("--concurrent-bwd", action="store_true", help="run dA on a side stream concurrent with dW (default)")
    ap.add_argument("--channelwise-tp", action="store_true",
                    help="SURVEY §8(f) row 2: channelwise tensor product (Alg. 2) + neighbour sum, forward + "
                         "backward (dY, dh, dR) per step on the bin's molecular graphs (degree 30); "
                         "metric symcon_tp_fwd_bwd_edges_per_s")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch eagerly (default at N=1: the step is replayed as a CUDA graph)")
    ap.add_argument("--graph-all", action="store_true",
                    help="also replay the step as a CUDA graph at N > 1 (device-side all-reduce epochs)")
    ap.add_argument("--double-backward", action="store_true",
                    help="force-training step (SURVEY §8(f) row 1): fwd + bwd + the double backward "
                         "(dB_bar, A_bar, W_bar of <uA, dA>) per step; metric symcon_fwd_bwd_bwd2_nodes_per_s")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                    help="arithmetic type of the plan (SURVEY §8(f) row 3: f64 = the paper's Float64 runs, "
                         "PAPER.md:1063; plain scalar DFMA kernels, NCCL all-reduce at N > 1)")
    ap.add_argument("--correlation", type=int, default=None, choices=[1, 2, 3, 4],
                    help="override the config's correlation order (4: reading s4b, plain scalar kernels)")
    a = ap.parse_args(argv)
    if a.capacity is None:
        a.capacity = DEFAULT_CAPACITY[a.config]
    return a


# ----------------------------------------------------------------------------- workload
def needs_l2_flush(step_input_bytes, pool_bytes, l2_bytes=L2_BYTES):
    """Timing rule: between timed steps either flush L2 or use inputs larger than L2. No flush when a
    step's own inputs exceed L2 or the pool of distinct bins cycled through is > 3x L2 (each step's
    inputs were evicted by the other bins' traffic); otherwise flush before every step."""
    return not (step_input_bytes > l2_bytes or pool_bytes > 3 * l2_bytes)


def shape_of(name, correlation=None):
    import dataclasses
    from synth.inputs import CONFIGS
    cfg = CONFIGS[name]
    return dataclasses.replace(cfg, correlation=correlation) if correlation else cfg


def fp64_lanes_per_sm_clk():
    """DFMA lane-ops per SM clock: measured by tools/probes/dfma_probe.cu (profiles/r02/dfma_probe.jsonl,
    best variant), else the nominal 64 (B200 FP64 = half the FP32 lane count)."""
    path = os.path.join(ROOT, "profiles", "r02", "dfma_probe.jsonl")
    if os.path.exists(path):
        vals = [json.loads(ln).get("dfma_per_sm_clk_median") for ln in open(path) if ln.startswith("{")]
        vals = [v for v in vals if v]
        if vals:
            return max(vals), "measured (tools/probes/dfma_probe.cu, profiles/r02/dfma_probe.jsonl)"
    return 64.0, "nominal (64 FP64 lanes per SM)"


def plan_bins(world, capacity=CAPACITY, seed=0):
    """Alg. 1 over the Table-2 manifest with libsymcon's C++ partitioner (GPU arm; same plan on
    every rank: deterministic)."""
    from synth.inputs import table2_sizes
    from paper_2504_10700_b200 import _lib
    sizes = table2_sizes(seed=seed)
    t0 = time.time()
    offs, ids = _lib.symcon_pack_balanced(sizes, capacity, world)
    return sizes, offs, ids, time.time() - t0


def plan_bins_oracle(world, capacity=CAPACITY, seed=0):
    """The same plan from the oracle's Alg. 1 (oracle/packing.py; reference arm -- no product code).
    tests/test_abi.py pins the two partitioners to identical bins."""
    from synth.inputs import table2_sizes
    from oracle.packing import create_balanced_batches
    sizes = table2_sizes(seed=seed)
    bins = create_balanced_batches([int(x) for x in sizes], capacity, world)
    offs = np.zeros(len(bins) + 1, np.int64)
    offs[1:] = np.cumsum([len(b) for b in bins])
    ids = np.array([g for b in bins for g in b], np.int64)
    return sizes, offs, ids


def bin_elements(sizes, offs, ids, b, n_elements):
    from synth.inputs import graph_elements
    g = ids[offs[b]:offs[b + 1]]
    return graph_elements(sizes[g], n_elements=n_elements, seed=0, salt=int(b))


def bin_inputs(cfg, sizes, offs, ids, b, q, rank, out_dim, n_lm, device):
    """(node_elem, A, dB) of bin b as pool entry q of `rank`: the same seeded values for the GPU arm
    and the oracle (synth draws on the CPU, then moves to `device`)."""
    import torch
    from synth.inputs import gen_A, gen_dB
    ne = torch.from_numpy(bin_elements(sizes, offs, ids, b, cfg.n_elements)).to(device)
    N = ne.numel()
    A = gen_A(N, cfg.channels, n_lm, device, seed=100 * q + rank)
    dB = gen_dB(N, out_dim, device, seed=100 * q + rank)
    return ne, A, dB


def molecule_batch(cfg, q, rank, out_dim, n_lm, device):
    """OFF-small (BASELINE.json configs[1]): a 20k-node batch of U[10, 100]-atom molecules with the organic
    element mix per node; pool entry q of `rank`. Returns (sizes, node_elem, A, dB)."""
    import torch
    from synth.inputs import gen_A, gen_dB, gen_node_elem, molecule_sizes
    sizes = np.array(molecule_sizes(OFF_BATCH_NODES, 10, 100, seed=100 * q + rank), dtype=np.int64)
    N = int(sizes.sum())
    ne = gen_node_elem(N, cfg.n_elements, cfg.elem_dist, device, seed=100 * q + rank)
    A = gen_A(N, cfg.channels, n_lm, device, seed=100 * q + rank)
    dB = gen_dB(N, out_dim, device, seed=100 * q + rank)
    return sizes, ne, A, dB


def edge_spread(sizes, offs, ids, world, steps):
    """Secondary balance metric (north_star: "balancing node and edge counts per GPU"): per step,
    max/mean over ranks of the bins' synthetic edge counts (degree min(30, n-1))."""
    from synth.inputs import graph_edges
    n_bins = len(offs) - 1
    worst, mean = 1.0, []
    for st in range(min(steps, n_bins // world)):
        e = [int(graph_edges(sizes[ids[offs[st * world + r]:offs[st * world + r + 1]]], EDGE_DEGREE).sum())
             for r in range(world)]
        m = max(float(np.mean(e)), 1.0)
        worst = max(worst, max(e) / m)
        mean.append(m)
    return {"edges_per_bin_mean": float(np.mean(mean)) if mean else 0.0, "edge_imbalance_max_over_mean": worst,
            "degree": f"min({EDGE_DEGREE}, n-1) per node"}


def alg_ops(sc):
    """Algorithmic FP32 lane-ops per (node, channel), per kernel and for the whole path, counted
    from the plan's tables. Each count is the smallest exact evaluation we know, so the
    roofline stays a bound ("If the builder finds an exact evaluation with fewer
    ops, lower the count to that"):
      fwd  = Horner per output slot (symcon_fwd_r): per slot, one FMA per degree-3 row
             (S_ab += c A_c), per prefix (T_a += A_b S_ab) and per first index (B += A_a T_a);
             the degree-1/2 coefficients enter as addends (705 at MP-medium)
      dA   = prefix products of degree-3 monomials + folded rows (g_j) + 2 per degree-3 monomial
             + 2 per prefix group + 1 per degree-1 monomial          (reverse of the prefix structure)
      dW   = reverse Horner per slot (symcon_bwd_dW_r): u_a = dB A_a per first index, q_ab = u_a A_b
             per prefix, one FMA per degree-3 row, one add per degree-1/2 row; a product that feeds
             only one add merges into an FMA (a prefix with only its degree-2 row, a first index with
             only its degree-1 row)
      path = fwd + dA + dW (the monomial-first forms, 888 / 888, are reported beside them)."""
    from paper_2504_10700_b200 import _lib
    if getattr(sc, "correlation", 3) == 4:
        return alg_ops_trie(sc)
    L, M, mono, col, val = _lib.symcon_plan_sym_table(sc.plan)
    rows = {(int(L[i]), int(M[i]), tuple(int(x) for x in mono[i])) for i in range(len(L))}
    monos = {r[2] for r in rows}
    deg = {m: sum(1 for x in m if x >= 0) for m in monos}
    prefixes = {m[:2] for m in monos if deg[m] >= 2}
    prefixes3 = {m[:2] for m in monos if deg[m] == 3}
    deg3 = sum(1 for m in monos if deg[m] == 3)
    deg1 = sum(1 for m in monos if deg[m] == 1)
    n_fold = len(rows)
    products = len(prefixes) + deg3
    fwd_mono = products + n_fold
    dW_mono = products + n_fold
    dA = len(prefixes3) + n_fold + 2 * deg3 + 2 * len(prefixes) + deg1
    # Horner / reverse-Horner counts per output slot (L, M)
    slots = {}
    for (Lr, Mr, m) in rows:
        slots.setdefault((Lr, Mr), []).append(m)
    fwd_h = dW_q = 0
    for ms in slots.values():
        r3 = [m for m in ms if m[2] >= 0]
        r2 = [m for m in ms if m[1] >= 0 and m[2] < 0]
        r1 = [m for m in ms if m[1] < 0]
        pre = {m[:2] for m in ms if m[1] >= 0}
        pre3 = {m[:2] for m in r3}
        firsts = {m[0] for m in ms}
        firsts_pre = {m[0] for m in ms if m[1] >= 0}
        fwd_h += len(r3) + len(pre) + len(firsts)
        dW_q += len(firsts) + len(pre) + len(r3) + len(r2) + len(r1) - len(pre - pre3) - len(firsts - firsts_pre)
    path = fwd_h + dA + dW_q
    path_mono = fwd_mono + (products + n_fold) + (n_fold + 2 * deg3 + 2 * len(prefixes) + deg1)
    # double backward (codegen symcon_bwd2 / symcon_bwd2_dW): per prefix p' (2 ops), p for degree-3
    # groups (1); per degree-3 monomial mono' (2) and, in the tile kernel, A_bar_c, h, h' (3); per
    # row one FMA into dB_bar (+ one into g for degree >= 2); per prefix group 2 (4 with h') FMAs
    # into A_bar_a, A_bar_b. W_bar: products as above + one FMA per row.
    rows1 = sum(1 for r in rows if deg[r[2]] == 1)
    p3 = len(prefixes3)
    bwd2 = rows1 + 2 * (n_fold - rows1) + 2 * len(prefixes) + p3 + 5 * deg3 + 4 * p3 + 2 * (len(prefixes) - p3)
    bwd2_dW = n_fold + 2 * len(prefixes) + p3 + 2 * deg3
    return {"fwd": fwd_h, "dA": dA, "dW": dW_q, "path": path, "bwd2": bwd2, "bwd2_dW": bwd2_dW,
            "fwd_monomial_first": fwd_mono, "dW_monomial_first": dW_mono, "path_monomial_first": path_mono,
            "n_fold": n_fold, "products": products, "prefixes": len(prefixes), "deg3_monomials": deg3,
            "n_sym": int(len(L))}


def alg_ops_trie(sc):
    """alg_ops for any degree (correlation 4), on the monomial prefix trie: forward = Horner per output
    slot = one FMA per node of the slot's trie; dW = the slot's reverse Horner = one product (or FMA) per
    trie node + one add per row sitting at an internal node; dA = the reverse of the global trie: one
    prefix product per internal node at depth >= 2, one op per folded row (g), 2 per node at depth >= 2
    (D_f += h P, h_parent += h A_f; at depth 2 the parent's share goes straight into D_a), 1 per degree-1
    monomial (D_a += g). At degree <= 3 these equal alg_ops' formulas exactly."""
    from paper_2504_10700_b200 import _lib
    L, M, mono, col, val = _lib.symcon_plan_sym_table(sc.plan, 4)
    rows = {(int(L[i]), int(M[i]), tuple(int(x) for x in mono[i] if x >= 0)) for i in range(len(L))}

    def trie(ms):
        nodes = {m[:d] for m in ms for d in range(1, len(m) + 1)}
        internal = {n[:-1] for n in nodes if len(n) >= 2}
        return nodes, internal
    slots = {}
    for (Lr, Mr, m) in rows:
        slots.setdefault((Lr, Mr), []).append(m)
    fwd = dW = 0
    for ms in slots.values():
        nodes, internal = trie(ms)
        fwd += len(nodes)
        dW += len(nodes) + sum(1 for m in ms if m in internal)
    monos = {r[2] for r in rows}
    nodes, internal = trie(monos)
    n_fold = len(rows)
    dA = sum(1 for n in internal if len(n) >= 2) + n_fold + 2 * sum(1 for n in nodes if len(n) >= 2) + \
        sum(1 for m in monos if len(m) == 1)
    return {"fwd": fwd, "dA": dA, "dW": dW, "path": fwd + dA + dW, "n_fold": n_fold, "monomials": len(monos),
            "trie_nodes": len(nodes), "n_sym": int(len(L)), "bwd2": 0, "bwd2_dW": 0,
            "note": "prefix-trie counts (alg_ops_trie); the plain scalar kernels execute the monomial-first forms"}


def path_roofline(cfg, sc, mean_nodes, path_ops, ms_step, dbl, sm_mhz=1965.0, esz=4, lanes=128):
    """Whole-step roofline: the step's algorithmic FP32 lane-ops at the ALU peak vs its
    algorithmic HBM bytes at the measured copy bandwidth (A read twice, dB, B and dA
    once per node-channel; the double backward adds uA, A, dB reads and dB_bar, A_bar writes)."""
    K = cfg.channels
    nlm = (cfg.lmax_in + 1) ** 2
    outc = sc.out_dim // K
    per = esz * (2 * nlm + outc + outc + nlm)
    if dbl:
        per += esz * (3 * nlm + outc + outc + nlm)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    t_alu = path_ops / (148 * lanes * sm_mhz * 1e6)
    t_hbm = per * mean_nodes * K / (hbm * 1e9)
    bound = "alu" if t_alu >= t_hbm else "hbm"
    out = {"bound": bound, "frac": max(t_alu, t_hbm) / (ms_step / 1e3), "t_alu_ms": t_alu * 1e3, "t_hbm_ms": t_hbm * 1e3,
           "bytes_per_node_channel": per, "sm_mhz": sm_mhz}
    if bound == "hbm":   # also against the spec HBM bandwidth (8 TB/s)
        out["frac_at_spec_hbm_8tbs"] = max(t_alu, per * mean_nodes * K / 8e12) / (ms_step / 1e3)
    return out


# ----------------------------------------------------------------------------- clocks
_CLOCK_CHILD = r"""
import json, select, sys, time
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
except Exception:
    try:
        print(json.dumps({"ready": None}), flush=True)
        sys.stdin.readline()
        print(json.dumps([]), flush=True)
    except Exception:
        pass
    sys.exit(0)
print(json.dumps({"ready": mx}), flush=True)
out = []
while not select.select([sys.stdin], [], [], 0)[0]:
    out.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
    time.sleep(float(sys.argv[2]))
sys.stdin.readline()
print(json.dumps(out), flush=True)
"""


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region by a separate sampler process
    (no GIL contention with the launching thread) polling NVML every ~2 ms from before the region
    starts; samples are kept if they fall inside [start, end] (marked by the caller) widened by 20 ms."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.samples = []          # (t, mhz, reasons)
        self.max_mhz = None
        self._p = None
        self.t0 = self.t1 = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        if os.environ.get("BENCH_CLOCK_RANK0") and int(os.environ.get("LOCAL_RANK", "0")) != 0:
            return self
        try:
            period = float(os.environ.get("BENCH_CLOCK_MS", "10")) / 1e3
            self._p = subprocess.Popen([sys.executable, "-c", _CLOCK_CHILD, str(self.index), str(period)], stdin=subprocess.PIPE,
                                       stdout=subprocess.PIPE, text=True)
            self.max_mhz = json.loads(self._p.stdout.readline())["ready"]
            time.sleep(0.02)
        except Exception:  # noqa: BLE001
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.02)
        try:
            self._p.stdin.write("stop\n")
            self._p.stdin.flush()
            self.samples = [tuple(x) for x in json.loads(self._p.stdout.readline())]
        except Exception:  # noqa: BLE001
            pass
        self._p.wait(timeout=10)

    def start(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def summary(self):
        t0 = (self.t0 or 0) - 0.02
        t1 = (self.t1 or time.time()) + 0.02
        win = [(m, r) for (t, m, r) in self.samples if t0 <= t <= t1]
        mx = self.max_mhz
        sm = [m for m, _ in win]
        reasons = sorted({name for _, r in win for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": mx, "reasons": reasons, "samples": len(sm), "source": f"nvml every {os.environ.get('BENCH_CLOCK_MS', '10')} ms (sampler process)"}


# ----------------------------------------------------------------------------- cpu oracle
def cpu_baseline(cfg, A, W, ne, dB, n_sample, seed=0, single_sample=512):
    """The oracle's plain C fp64 loop (never tuned) on a bounded sample of the workload: all cores
    of the affinity mask, and one thread on a smaller sample."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    oc = OracleC(Problem(cfg.lmax_in, cfg.correlation, cfg.out_L))
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(A.shape[0], min(n_sample, A.shape[0]), replace=False))
    import torch
    ti = torch.from_numpy(idx).to(A.device)
    hA, hne, hdB = A[ti].cpu().numpy(), ne[ti].cpu().numpy(), dB[ti].cpu().numpy()
    hW = W.cpu().numpy()
    t0 = time.time()
    oc.forward(hA, hW, hne)
    oc.backward(hA, hW, hne, hdB)
    dt = time.time() - t0
    cores = oc.threads()
    n1 = min(single_sample, len(idx))
    oc.lib.oracle_set_threads(1)
    t1 = time.time()
    oc.forward(hA[:n1], hW, hne[:n1])
    oc.backward(hA[:n1], hW, hne[:n1], hdB[:n1])
    dt1 = time.time() - t1
    oc.lib.oracle_set_threads(cores)
    import platform
    model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")), platform.processor())
    return {"value": len(idx) / dt, "unit": "nodes/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(idx)} random nodes of one {A.shape[0]}-node bin, fwd+bwd (B, dA, dW), fp64 C/OpenMP loop "
                      f"over {oc.n_terms} raw U terms per (node, channel), {dt:.1f} s",
            "single_thread": {"value": n1 / dt1, "unit": "nodes/s", "cores": 1, "sample": f"first {n1} nodes of the sample, {dt1:.1f} s"},
            "cpu_model": model}


def run_reference(args):
    """--impl reference: the oracle (oracle/ only: Alg. 1 from oracle/packing.py, the plain C fp64
    evaluator) on the host cores. Same workload as the GPU arm's first pool entry on rank 0: the same
    Alg. 1 bin, the same seeded node elements, A and dB; each step a bounded sample of its nodes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.inputs import gen_W
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    cfg = shape_of(args.config, args.correlation)
    prob = Problem(cfg.lmax_in, cfg.correlation, cfg.out_L)
    oc = OracleC(prob)
    world = max(args.gpus, 1)
    t0 = time.time()
    n_lm = (cfg.lmax_in + 1) ** 2
    if args.capacity is None:   # off_small: the GPU arm's first molecule batch of rank 0
        _, ne_t, A_t, dB_t = molecule_batch(cfg, 0, 0, prob.out_dim(cfg.channels), n_lm, "cpu")
    else:
        sizes, offs, ids = plan_bins_oracle(world, args.capacity)
        b = 0   # pool entry 0 of rank 0 = step 0's bin of rank 0
        ne_t, A_t, dB_t = bin_inputs(cfg, sizes, offs, ids, b, 0, 0, prob.out_dim(cfg.channels), n_lm, "cpu")
    t_pack = time.time() - t0
    ne_full, A_full, dB_full = ne_t.numpy(), A_t.numpy(), dB_t.numpy()
    n_bin = len(ne_full)
    W = gen_W(cfg.n_elements, prob.block_sizes(), cfg.channels, "cpu").numpy()
    per_step = max(64, min(n_bin, args.cpu_sample // 8))
    perm = np.random.default_rng(0).permutation(n_bin)

    def sample(q):
        idx = np.sort(perm[(q * per_step) % n_bin:][:per_step])
        return A_full[idx], ne_full[idx], dB_full[idx]
    for q in range(args.warmup):
        a, e, d = sample(q)
        oc.forward(a[:16], W, e[:16])
    t0 = time.time()
    for q in range(args.steps):
        a, e, d = sample(q)
        oc.forward(a, W, e)
        oc.backward(a, W, e, d)
    dt = time.time() - t0
    v = per_step * args.steps / dt
    out = {"impl": "reference", "metric": "symcon_fwd_bwd_nodes_per_s", "value": v, "unit": "nodes/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args, cfg, n_bin),
           "same_config": True,
           "cpu_baseline": {"value": v, "unit": "nodes/s", "cores": oc.threads(), "kind": "oracle",
                            "sample": f"{per_step} nodes per step (seeded permutation of batch 0, the GPU arm's pool entry 0 "
                                      f"on rank 0: same batch, node elements, A, dB, W) x {args.steps} steps"},
           "alg1_pack_s": round(t_pack, 3), "oracle_only": "oracle/packing.py + oracle/csrc/oracle_eval.c; libsymcon not loaded",
           "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_config(args, cfg, nodes_per_bin):
    return {"workload": f"{args.config}_dp_step" + ("_double_backward" if args.double_backward else "")
                        + ("" if args.capacity == DEFAULT_CAPACITY[args.config] else f"_C{args.capacity}")
                        + (f"_corr{args.correlation}" if args.correlation else "")
                        + ("_f64" if args.dtype == "f64" else ""),
            "batch": ("20k-node batches of U[10,100]-atom molecules, organic element mix" if args.capacity is None else
                      f"Alg. 1 bins of the Table-2 manifest, capacity {args.capacity} nodes"),
            "model": "MACE symmetric contraction", "channels": cfg.channels,
            "out": "+".join(f"{cfg.channels}x{L}{'e' if L % 2 == 0 else 'o'}" for L in cfg.out_L),
            "lmax_in": cfg.lmax_in, "correlation": cfg.correlation, "elements": cfg.n_elements,
            "capacity_nodes": args.capacity, "nodes_bin0": int(nodes_per_bin)}


# ----------------------------------------------------------------------------- the timed step
class TimedStep:
    """The step bench.py times, on this rank: a pool of `pool` distinct Alg. 1 bins resident in
    HBM (bin of step q % n_steps for this rank), W replicated, one DataParallelContraction
    (dW on the main stream, dA concurrently on a side stream sharing the workspace, reuse hints
    after the forward, and for N > 1 the dW all-reduce), optionally replayed from one CUDA graph
    per pool entry. tests/test_gpu_timed_step.py drives this very object and checks its outputs
    against the oracle."""

    def __init__(self, config="mp_medium", capacity=CAPACITY, world=1, rank=0, device=0, pool=POOL,
                 double_backward=False, allreduce="peer", peer_algo=0, overlap=True, concurrent_bwd=None,
                 dtype="f32", correlation=None):
        import torch
        from paper_2504_10700_b200.ops import SymmetricContraction
        from paper_2504_10700_b200.dist import BinPackedShards, DataParallelContraction
        from synth.inputs import gen_A, gen_W, table2_sizes
        self.torch = torch
        self.cfg = cfg = shape_of(config, correlation)
        self.dev = dev = torch.device("cuda", device)
        self.world, self.rank, self.double_backward = world, rank, double_backward
        self.dtype = tdt = torch.float64 if dtype == "f64" else torch.float32
        if tdt == torch.float64:
            allreduce = "nccl"     # the peer all-reduce kernel is fp32
        self.sc = sc = SymmetricContraction(cfg.lmax_in, cfg.correlation, cfg.out_L, cfg.n_elements, cfg.channels,
                                            device=device, dtype=tdt)
        self.capacity = capacity
        self.pool, self.uA, self.mol_sizes = [], {}, []
        t0 = time.time()
        if capacity is not None:
            self.sizes = table2_sizes(seed=0)
            self.shards = BinPackedShards(self.sizes, capacity, world, rank)
        else:
            self.sizes = self.shards = None
        self.t_pack = time.time() - t0
        for q in range(pool):
            if capacity is not None:
                b = self.shards.bin_of(q % self.shards.n_steps)
                ne, A, dB = bin_inputs(cfg, self.sizes, self.shards.offsets, self.shards.ids, b, q, rank, sc.out_dim,
                                       sc.n_lm, dev)
            else:
                b = q
                msz, ne, A, dB = molecule_batch(cfg, q, rank, sc.out_dim, sc.n_lm, dev)
                self.mol_sizes.append(msz)
            N = ne.numel()
            A, dB = A.to(tdt), dB.to(tdt)      # same seeded values (drawn in fp32) in the plan's dtype
            B = torch.empty((N, sc.out_dim), device=dev, dtype=tdt)
            dA = torch.empty_like(A)
            self.pool.append((b, N, A, ne, dB, B, dA))
            if double_backward:
                self.uA[q] = gen_A(N, cfg.channels, sc.n_lm, dev, seed=100 * q + rank + 7)
        self.imbalance = (max(self.shards.step_imbalance(q % self.shards.n_steps) for q in range(pool))
                          if self.shards is not None else 1.0)
        self.W = gen_W(cfg.n_elements, sc.block_sizes(), cfg.channels, dev).to(tdt)
        if world > 1:
            import torch.distributed as dist
            dist.broadcast(self.W, 0)
        self.dW = torch.empty_like(self.W)
        for q in range(pool):
            sc.workspace(self.pool[q][1])
        self.dp = DataParallelContraction(sc, overlap=overlap, concurrent_bwd=concurrent_bwd, allreduce=allreduce,
                                          peer_algo=peer_algo)
        self.graphs = None
        self.outputs = {}   # q -> (B, dA, dW[, W_bar]) of the last call for pool entry q (views; dW shared)

    def eager(self, q, runner=None):
        dp = runner or self.dp
        b, N, A, ne, dB, B, dA = self.pool[q % len(self.pool)]
        dp.forward(A, self.W, ne, B=B)
        dp.backward(A, self.W, ne, dB, dA=dA, dW=self.dW)
        if self.double_backward:
            dp.backward2(A, self.W, ne, dB, self.uA[q % len(self.pool)])
        return N

    def capture(self):
        """One CUDA graph per pool entry (the whole step); launch counts taken at capture."""
        torch = self.torch
        self.graphs, self.per_step = [], []
        for q in range(len(self.pool)):
            g = torch.cuda.CUDAGraph()
            n0 = self.dp.launches
            with torch.cuda.graph(g):
                self.eager(q)
            self.per_step.append(self.dp.launches - n0)
            self.graphs.append(g)
        torch.cuda.synchronize()
        for q in range(len(self.pool)):   # a whole cycle, so the timed replays continue the buffer alternation
            self.step(q)
        torch.cuda.synchronize()

    def step(self, q):
        if self.graphs is None:
            return self.eager(q)
        self.graphs[q % len(self.pool)].replay()
        self.dp.launches += self.per_step[q % len(self.pool)]
        for r in (self.dp._peer, self.dp._peer2):
            if r is not None:
                # graph q was captured with buffer parity q % 2; keep eager calls alternating too
                r.parity = (q + 1) % 2
        return self.pool[q % len(self.pool)][1]


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != max(args.gpus, 1) and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2504_10700_b200 import _lib
    from paper_2504_10700_b200.dist import DataParallelContraction
    cfg = shape_of(args.config, args.correlation)
    conc = False if args.sequential_bwd else (True if args.concurrent_bwd else None)
    ts = TimedStep(args.config, args.capacity, world, rank, local, POOL, args.double_backward, args.allreduce,
                   args.peer_algo, not args.no_overlap, conc, args.dtype, args.correlation)
    sc, dp, W, dW, pool = ts.sc, ts.dp, ts.W, ts.dW, ts.pool
    for q in range(args.warmup):
        ts.eager(q)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    assert s == 0, (s, bad)
    use_graph = (world == 1 or args.graph_all) and not args.no_graph
    if use_graph:
        ts.capture()
    dp.check()   # raises if a peer all-reduce barrier timed out (dW / W_bar then NaN)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.symcon_profile_reset(sc.plan)
    dp.launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nodes = 0
    # L2 hygiene: a step's inputs larger than L2, or a pool of distinct bins much larger than L2, need no
    # flush; otherwise (C = 3,072: 25 MB per bin) L2 is flushed before every timed step by a 256 MB memset
    # outside that step's own event pair, and the step times are summed
    step_in = max(x[2].nbytes + x[3].nbytes + x[4].nbytes for x in pool)
    pool_bytes = sum(x[2].nbytes + x[3].nbytes + x[4].nbytes + x[5].nbytes + x[6].nbytes for x in pool)
    flush = needs_l2_flush(step_in, pool_bytes)
    scratch = torch.empty(int(2 * L2_BYTES), dtype=torch.uint8, device=dev) if flush else None
    # per-step event pairs (median / min per step beside the mean the line's value uses)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # ranks enter the timed region together (the sampler start-up takes a variable fraction
        # of a second per rank; without this barrier the first rank's wait is charged to the others)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.start()
        e0.record()
        for q in range(args.steps):
            if flush:
                scratch.zero_()
            evs[q][0].record()
            nodes += ts.step(q)
            evs[q][1].record()
        e1.record()
        torch.cuda.synchronize()
        clk.end()
    if world > 1:
        dist.barrier()
    dp.check()
    step_ms = sorted(a.elapsed_time(b) for a, b in evs)
    ms = sum(step_ms) if flush else e0.elapsed_time(e1)
    l2_note = (f"L2 flushed before every timed step (256 MB memset outside the step's CUDA-event pair; pool of "
               f"{len(pool)} bins = {pool_bytes / 1e6:.0f} MB, step inputs {step_in / 1e6:.0f} MB)" if flush else
               f"no flush: step inputs {step_in / 1e6:.0f} MB (A, node_elem, dB) and a pool of {len(pool)} distinct bins "
               f"({pool_bytes / 1e6:.0f} MB) cycled, vs 126 MB of L2")
    launches_timed = dp.launches
    # per-kernel times for the roofline: a separate pass with the kernels back to back on one
    # stream (the throughput region above overlaps dW and dA, which would blur each kernel's time)
    _lib.symcon_profile_enable(sc.plan, 1)
    _lib.symcon_profile_reset(sc.plan)
    seq = DataParallelContraction(sc, overlap=not args.no_overlap, concurrent_bwd=False, allreduce="nccl")
    for q in range(args.steps):
        ts.eager(q, runner=seq)
    torch.cuda.synchronize()
    prof = _lib.symcon_profile_read(sc.plan)
    _lib.symcon_profile_enable(sc.plan, 0)
    # the all-reduce alone (N > 1): device time per call on the main stream
    ar_ms = None
    if world > 1 and dp._peer is not None:
        dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(10):
            dp._peer.allreduce(dW, torch.cuda.current_stream().cuda_stream)
        a1.record()
        torch.cuda.synchronize()
        dp.check()
        ar_ms = a0.elapsed_time(a1) / 10
    t = torch.tensor([ms, nodes], dtype=torch.float64, device=dev)
    if world > 1:
        tt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tt, t)
        ms_max = max(float(x[0]) for x in tt)
        nodes_all = sum(float(x[1]) for x in tt)
        per_rank_ms = [round(float(x[0]) / args.steps, 4) for x in tt]
    else:
        ms_max, nodes_all = ms, float(nodes)
        per_rank_ms = [round(ms / args.steps, 4)]
    value = nodes_all / (ms_max / 1e3)

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    b, N, A, ne, dB, B, dA = pool[0]
    hA, hne, hdB = A.cpu().pin_memory(), ne.cpu().pin_memory(), dB.cpu().pin_memory()
    hdW = torch.empty(W.shape, dtype=W.dtype).pin_memory()
    hU = ts.uA[0].cpu().pin_memory() if args.double_backward else None
    dA2 = torch.empty_like(A)
    # two device input sets: the host->device copy of step s+1 (copy stream) overlaps the compute
    # of step s; every step still copies its own inputs and reads its dW back inside the region
    sets = [dict(A=torch.empty_like(A), ne=torch.empty_like(ne), dB=torch.empty_like(dB),
                 U=torch.empty_like(A) if args.double_backward else None) for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def e2e_copy(slot):
        x = sets[slot]
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[slot])
            x["A"].copy_(hA, non_blocking=True)
            x["ne"].copy_(hne, non_blocking=True)
            x["dB"].copy_(hdB, non_blocking=True)
            if args.double_backward:
                x["U"].copy_(hU, non_blocking=True)
            copied[slot].record(copy_stream)

    def e2e_run(n_steps):
        main = torch.cuda.current_stream(dev)
        e2e_copy(0)
        for q in range(n_steps):
            x = sets[q % 2]
            main.wait_event(copied[q % 2])
            if q + 1 < n_steps:
                e2e_copy((q + 1) % 2)
            dp.forward(x["A"], W, x["ne"], B=B)
            dp.backward(x["A"], W, x["ne"], x["dB"], dA=dA2, dW=dW)
            hdW.copy_(dW, non_blocking=True)
            if args.double_backward:
                _, _, Wb = dp.backward2(x["A"], W, x["ne"], x["dB"], x["U"])
                hdW.copy_(Wb, non_blocking=True)
            consumed[q % 2].record(main)

    e2e_steps = max(4, min(args.steps, 10))
    e2e_run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    e2e_run(e2e_steps)
    f1.record()
    torch.cuda.synchronize()
    dp.check()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    t2 = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = N * world / (float(t2[0]) / 1e3)
    esz = A.element_size()
    h2d = hA.numel() * esz + hne.numel() * 4 + hdB.numel() * esz + (hU.numel() * esz if hU is not None else 0)
    d2h = hdW.numel() * esz * (2 if args.double_backward else 1)

    if rank == 0:
        ops = alg_ops(sc)
        K = cfg.channels
        clocks = clk.summary()
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        lanes, lanes_src = (fp64_lanes_per_sm_clk() if args.dtype == "f64" else (128.0, "148 SMs x 128 FP32 lanes"))
        peak_alu = 148 * lanes * sm_mhz * 1e6 / 1e12          # T lane-ops/s at the sampled clock
        mean_nodes = nodes / args.steps
        roof = kernel_roofline(args, cfg, sc, ops, prof, mean_nodes, peak_alu, sm_mhz, esz, lanes, lanes_src)
        path_ops = (ops["path"] + (ops["bwd2"] + ops["bwd2_dW"] if args.double_backward else 0)) * mean_nodes * K
        kernels = {k: {"launches": v[0], "avg_ms": v[1] / max(v[0], 1)} for k, v in prof.items()}
        ms_step = ms_max / args.steps
        ksum = sum(v["avg_ms"] * v["launches"] for v in kernels.values()) / args.steps
        config = workload_config(args, cfg, pool[0][1])
        config.update({"bins": ts.shards.n_bins if ts.shards is not None else None, "global_batch": int(nodes_all / args.steps),
                       "step_imbalance_max_over_mean": round(ts.imbalance, 5),
                       "dW_allreduce": ({"peer": f"libsymcon NVLink peer-memory kernel (algo {dp._peer.algo if dp._peer else args.peer_algo}: "
                                                 "0 auto, 1 one-shot, 2 two-shot), dA concurrent",
                                         "nccl": "NCCL on a communication stream"}[dp.allreduce] if world > 1 else None),
                       "seq_len": None, "parallelism": f"dp{world}",
                       "l2": l2_note,
                       "alg1_pack_s": round(ts.t_pack, 3), "cuda_graph": use_graph})
        out = {
            "metric": "symcon_fwd_bwd_bwd2_nodes_per_s" if args.double_backward else "symcon_fwd_bwd_nodes_per_s",
            "value": value, "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": config,
            "per_gpu_nodes_per_s": value / world,
            "per_rank_ms_per_step": per_rank_ms,
            "step_ms_rank0": {"median": statistics.median(step_ms), "min": step_ms[0], "max": step_ms[-1],
                              "note": "per-step CUDA-event pairs on rank 0 (the value uses the whole timed region)"},
            "edge_balance": (edge_spread(ts.sizes, ts.shards.offsets, ts.shards.ids, world, POOL) if ts.shards is not None
                             else {"note": "one molecule batch per rank (no Alg. 1 bins)"}),
            "path_tops": path_ops / (ms_step / 1e3) / 1e12,
            "path_frac_of_alu_peak": path_ops / (ms_step / 1e3) / 1e12 / peak_alu,
            "path_roofline": path_roofline(cfg, sc, mean_nodes, path_ops, ms_step, args.double_backward, sm_mhz, esz, lanes),
            "roofline": roof, "kernels": kernels, "alg_ops_per_node_channel": ops,
            "step_breakdown_ms": {"step": ms_step, "kernels_back_to_back": ksum,
                                  "allreduce_alone": ar_ms,
                                  "note": "kernels_back_to_back = sum of per-launch-group CUDA-event times from the "
                                          "sequential pass (dW and dA not overlapped); allreduce_alone = one peer "
                                          "all-reduce call timed alone"},
            "clocks": clocks, "gpu_launches": launches_timed,
            "kernel_timing": "per-kernel CUDA events from a separate pass of the same steps with dW and dA back to back",
            "e2e": {"value": e2e_value, "unit": "nodes/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "note": "H2D A+node_elem+dB from pinned host, D2H dW, per step through SymmetricContraction; "
                            "the copy of step s+1 (copy stream) overlaps the compute of step s"},
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, A, W, ne, dB, args.cpu_sample)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def kernel_roofline(args, cfg, sc, ops, prof, mean_nodes, peak_alu, sm_mhz, esz=4, lanes=128.0, lanes_src=None):
    """roofline of the dominant kernel (by measured time): its algorithmic ops (or bytes) per launch
    / its average CUDA-event launch time, against the FP32 peak at the sampled SM clock (or the
    measured HBM copy bandwidth), whichever binds it."""
    if not prof:
        return None
    kern = max(prof, key=lambda k: prof[k][1])
    cnt, tot_ms = prof[kern]
    avg_ms = tot_ms / max(cnt, 1)
    K = cfg.channels
    per_nc = {"symcon_fwd": ops["fwd"], "symcon_bwd_dA": ops["dA"], "symcon_bwd_dW": ops["dW"],
              "symcon_bwd2": ops["bwd2"], "symcon_bwd2_dW": ops["bwd2_dW"]}.get(kern)
    if not per_nc:
        return {"kernel": kern, "avg_launch_ms": avg_ms}
    achieved = per_nc * mean_nodes * K / (avg_ms / 1e3) / 1e12   # T lane-ops/s
    nlm = (cfg.lmax_in + 1) ** 2
    outc = sc.out_dim // K
    alg_b = {"symcon_fwd": esz * (nlm + outc), "symcon_bwd_dA": esz * (2 * nlm + outc),
             "symcon_bwd_dW": esz * (nlm + outc), "symcon_bwd2": esz * (4 * nlm + 2 * outc),
             "symcon_bwd2_dW": esz * (2 * nlm + outc)}[kern] * mean_nodes * K
    traffic, tsrc = None, None
    for tpath in (os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json"),):
        if (os.path.exists(tpath) and args.config == "mp_medium" and args.capacity == DEFAULT_CAPACITY["mp_medium"]
                and args.dtype == "f32" and not args.correlation):
            tj = json.load(open(tpath))
            rec = tj["kernels"].get(kern)
            if rec:
                traffic = rec["dram_bytes_read"] + rec["dram_bytes_write"]
                tsrc = tj["source"]
    hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    t_alu = per_nc * mean_nodes * K / (peak_alu * 1e12)
    t_hbm = alg_b / (hbm_peak * 1e9)
    common = {"kernel": kern, "traffic": traffic, "traffic_source": tsrc, "algorithmic_bytes": alg_b,
              "avg_launch_ms": avg_ms, "ops_per_node_channel": per_nc}
    if t_hbm > t_alu:
        gbs = alg_b / (avg_ms / 1e3) / 1e9
        return dict(common, bound="hbm", achieved=gbs, peak=hbm_peak, unit="GB/s", frac=gbs / hbm_peak,
                    alu_tops=achieved, alu_frac=achieved / peak_alu,
                    peak_derivation="MEASURED_PEAKS.json hbm_gbs (copy bandwidth)")
    prec = "fp64 DFMA" if esz == 8 else "fp32 FMA"
    return dict(common, bound="alu", achieved=achieved, peak=peak_alu, unit=f"Tops/s ({prec} lane-ops)",
                frac=achieved / peak_alu, hbm_gbs=alg_b / (avg_ms / 1e3) / 1e9,
                frac_at_max_clock=achieved / (148 * lanes * 1.965e-3),
                peak_derivation=f"148 SMs x {lanes:g} lanes per clock ({lanes_src or 'FP32'}) x {sm_mhz:.0f} MHz (median SM "
                                "clock sampled during the timed region; DESIGN.md §7)")


# ----------------------------------------------------------------------------- channelwise TP
def tp_bytes(N, E, K, P, NH, NY, NOUT):
    """Algorithmic HBM bytes of one TP step: every input read once, every output
    written once (h, dA per node; R, Y per edge; no intermediate)."""
    fwd = 4 * (E * K * P + N * K * NH + E * NY + N * K * NOUT) + 8 * E
    bwd = 4 * (E * K * P + N * K * NH + E * NY + N * K * NOUT) + 8 * E + 4 * (E * NY + N * K * NH + E * K * P)
    return fwd, bwd


def run_tp(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2504_10700_b200.ops import ChannelwiseTP
    from paper_2504_10700_b200.dist import BinPackedShards
    from synth.inputs import table2_sizes, gen_tp_graph, gen_tp_inputs
    K, LMAX_Y, HIDDEN, LMAX_OUT, DEG = 128, 3, (0, 1), 3, 30
    tp = ChannelwiseTP(LMAX_Y, HIDDEN, LMAX_OUT, K, device=local)
    sizes = table2_sizes(seed=0)
    shards = BinPackedShards(sizes, CAPACITY, world, rank)
    pool = []
    for q in range(2):
        b = shards.bin_of(q % shards.n_steps)
        snd, rcv = gen_tp_graph(sizes[shards.graphs(q % shards.n_steps)], DEG, seed=b)
        N, E = int(sizes[shards.graphs(q % shards.n_steps)].sum()), len(snd)
        Y, h, R = gen_tp_inputs(N, E, K, tp.n_y, tp.n_h, tp.n_paths, dev, seed=100 * q + rank)
        dA = torch.randn((N, K, tp.n_out), generator=torch.Generator(dev).manual_seed(q), device=dev)
        pool.append(dict(N=N, E=E, Y=Y, h=h, R=R, s=torch.from_numpy(snd).to(dev), r=torch.from_numpy(rcv).to(dev),
                         dA=dA, A=torch.empty((N, K, tp.n_out), device=dev), dY=torch.empty_like(Y),
                         dh=torch.empty_like(h), dR=torch.empty_like(R)))
    tp.workspace(max(x["N"] for x in pool), max(x["E"] for x in pool))
    from paper_2504_10700_b200 import _lib
    launches = [0]

    def step(q, ev=None):
        x = pool[q % len(pool)]
        st = torch.cuda.current_stream(dev).cuda_stream
        ws = tp._ws
        if ev:
            ev[0].record()
        _lib.symcon_tp_forward(tp.plan, x["N"], x["E"], x["Y"].data_ptr(), x["h"].data_ptr(), x["R"].data_ptr(),
                               x["s"].data_ptr(), x["r"].data_ptr(), x["A"].data_ptr(), ws.data_ptr(), ws.numel(), st)
        launches[0] += tp.last_launch_count()
        if ev:
            ev[1].record()
        _lib.symcon_tp_backward(tp.plan, x["N"], x["E"], x["Y"].data_ptr(), x["h"].data_ptr(), x["R"].data_ptr(),
                                x["s"].data_ptr(), x["r"].data_ptr(), x["dA"].data_ptr(), x["dY"].data_ptr(),
                                x["dh"].data_ptr(), x["dR"].data_ptr(), ws.data_ptr(), ws.numel(), st,
                                _lib.SYMCON_TP_REUSE_GRAPH)   # the step's graph, built by its forward
        launches[0] += tp.last_launch_count()
        if ev:
            ev[2].record()
        return x["N"], x["E"]

    for q in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    st_, bad = tp.check_device_error()
    assert st_ == 0, (st_, bad)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nodes = edges = 0
    with ClockSampler(local) as clk:
        # ranks enter the timed region together (the sampler start-up takes a variable fraction
        # of a second per rank; without this barrier the first rank's wait is charged to the others)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.start()
        e0.record()
        for q in range(args.steps):
            n_, e_ = step(q)
            nodes += n_
            edges += e_
        e1.record()
        torch.cuda.synchronize()
        clk.end()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    n_launch = launches[0]
    # per-phase times (fwd, bwd) from a separate pass of the same steps
    tf = tb = 0.0
    for q in range(args.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        step(q, ev)
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    t = torch.tensor([ms, nodes, edges], dtype=torch.float64, device=dev)
    if world > 1:
        tt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tt, t)
        ms_max = max(float(x[0]) for x in tt)
        edges_all = sum(float(x[2]) for x in tt)
        nodes_all = sum(float(x[1]) for x in tt)
    else:
        ms_max, edges_all, nodes_all = ms, float(edges), float(nodes)
    value = edges_all / (ms_max / 1e3)
    # e2e: host inputs (pinned) copied in, gradients copied out, every step
    x = pool[0]
    hY, hh, hR, hs, hr, hdA = (x[k].cpu().pin_memory() for k in ("Y", "h", "R", "s", "r", "dA"))
    hdR = torch.empty(x["R"].shape).pin_memory()
    hdh = torch.empty(x["h"].shape).pin_memory()
    hdY = torch.empty(x["Y"].shape).pin_memory()
    dev_bufs = {k: torch.empty_like(x[k]) for k in ("Y", "h", "R", "s", "r", "dA")}

    def e2e():
        for k, hsrc in zip(("Y", "h", "R", "s", "r", "dA"), (hY, hh, hR, hs, hr, hdA)):
            dev_bufs[k].copy_(hsrc, non_blocking=True)
        tp.forward_raw(dev_bufs["Y"], dev_bufs["h"], dev_bufs["R"], dev_bufs["s"], dev_bufs["r"], A=x["A"])
        dY, dh, dR = tp.backward_raw(dev_bufs["Y"], dev_bufs["h"], dev_bufs["R"], dev_bufs["s"], dev_bufs["r"],
                                     dev_bufs["dA"], reuse=True)
        hdY.copy_(dY, non_blocking=True)
        hdh.copy_(dh, non_blocking=True)
        hdR.copy_(dR, non_blocking=True)

    e2e()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne2e = 3
    f0.record()
    for _ in range(ne2e):
        e2e()
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / ne2e
    if rank == 0:
        P, NH, NY, NOUT = tp.n_paths, tp.n_h, tp.n_y, tp.n_out
        fb, bb = tp_bytes(x["N"], x["E"], K, P, NH, NY, NOUT)
        mean_e = edges / args.steps
        mean_n = nodes / args.steps
        fb, bb = tp_bytes(mean_n, mean_e, K, P, NH, NY, NOUT)
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
        avg_f, avg_b = tf / args.steps, tb / args.steps
        dom = ("symcon_tp_bwd", bb, avg_b) if avg_b >= avg_f else ("symcon_tp_fwd", fb, avg_f)
        achieved = dom[1] / (dom[2] / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "r01", "ncu_tp_traffic.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            rec = tj.get("kernels", {}).get(dom[0])
            if rec:
                traffic = rec["dram_bytes_read"] + rec["dram_bytes_write"]
        h2d = sum(t.numel() * t.element_size() for t in (hY, hh, hR, hs, hr, hdA))
        d2h = sum(t.numel() * t.element_size() for t in (hdY, hdh, hdR))
        cpu = None
        if not args.no_cpu_baseline:
            from oracle.tp import TPProblem, forward as tpf, backward as tpb
            prob = TPProblem(LMAX_Y, HIDDEN, LMAX_OUT)
            hs_np, hr_np = x["s"].cpu().numpy(), x["r"].cpu().numpy()
            sel = np.nonzero(hr_np < 800)[0]            # edges into the first 800 nodes
            te = torch.from_numpy(sel).to(dev)
            cY, cR = x["Y"][te].cpu().numpy(), x["R"][te].cpu().numpy()
            ch_, cdA = x["h"].cpu().numpy(), x["dA"].cpu().numpy()
            t0 = time.time()
            tpf(prob, cY, ch_, cR, hs_np[sel], hr_np[sel], x["N"])
            tpb(prob, cY, ch_, cR, hs_np[sel], hr_np[sel], x["N"], cdA)
            dt = time.time() - t0
            cpu = {"value": len(sel) / dt, "unit": "edges/s", "cores": 1, "kind": "oracle",
                   "sample": f"{len(sel)} edges (into the first 800 nodes of one bin), fwd + bwd, numpy fp64 oracle "
                             f"(oracle/tp.py), {dt:.1f} s"}
        out = {
            "metric": "symcon_tp_fwd_bwd_edges_per_s", "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "channelwise_tp_mp_layer2_dp_step", "channels": K, "lmax_y": LMAX_Y,
                       "hidden": "+".join(f"{K}x{l}{'e' if l % 2 == 0 else 'o'}" for l in HIDDEN),
                       "lmax_out": LMAX_OUT, "paths": P, "degree": DEG, "capacity_nodes": CAPACITY,
                       "nodes_per_step": int(nodes_all / args.steps), "edges_per_step": int(edges_all / args.steps),
                       "parallelism": f"dp{world}", "l2": "inputs > L2 (R 7.5 GB per bin), 2-bin pool"},
            "nodes_per_s": nodes_all / (ms_max / 1e3),
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes": dom[1],
                         "avg_launch_ms": dom[2],
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                         "note": "time of the launch group (CSR + kernel [+ dh reduce]) from CUDA events"},
            "phases_ms": {"fwd": avg_f, "bwd": avg_b},
            "clocks": clk.summary(), "gpu_launches": n_launch,
            "e2e": {"value": x["E"] / (e2e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "note": "pinned host Y, h, R, edges, dA in; dY, dh, dR out"},
        }
        if cpu:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.channelwise_tp:
        run_tp(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

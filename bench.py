"""Benchmark: symmetric-contraction fwd+bwd nodes/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config mp_medium]

A step is one pass of the whole hot path over one bin of molecular graphs per GPU:
element bucketing, W-fold, forward B, backward dW (S partials + fixed-order reduction) and
dA, and — for N > 1 — the NCCL all-reduce of dW. Workload (SURVEY.md §8(d) config 5 at the
MP-medium shape): the 2,650,823-graph Table-2 manifest packed by Alg. 1 (C++ partitioner,
capacity 50,000 nodes, M = multiple of N bins), bin s*N + r on rank r at step s; 128
channels, 0e+1o output, lmax 3, correlation 3, 89 elements (1-4 Zipf elements per graph).
Inputs for the timed steps are resident in HBM before timing; A alone is 410 MB per bin,
larger than L2, and a pool of distinct bins is cycled, so no L2 flush is needed.

One JSON line on rank 0. `roofline` reports the dominant kernel (FP32 ALU bound), its
per-launch CUDA-event time measured by libsymcon's launch timer inside the timed region.
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
POOL = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mp_medium", choices=["off_small", "mp_medium", "large"])
    ap.add_argument("--cpu-sample", type=int, default=32768, help="nodes in the oracle's bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="all-reduce dW after dA instead of overlapping")
    ap.add_argument("--allreduce", default="peer", choices=["peer", "nccl"],
                    help="N > 1: dW all-reduce by libsymcon's NVLink peer-memory kernel (default) or NCCL")
    ap.add_argument("--sequential-bwd", action="store_true", help="run the dW and dA kernels back to back on one stream")
    ap.add_argument("--concurrent-bwd", action="store_true", help="run dA on a side stream concurrent with dW (default at N=1)")
    ap.add_argument("--channelwise-tp", action="store_true",
                    help="SURVEY §8(f) row 2: channelwise tensor product (Alg. 2) + neighbour sum, forward + "
                         "backward (dY, dh, dR) per step on the bin's molecular graphs (degree 30); "
                         "metric symcon_tp_fwd_bwd_edges_per_s")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch eagerly (default at N=1: the step is replayed as a CUDA graph; N>1 always eager "
                         "because the peer all-reduce takes a fresh barrier epoch per call)")
    ap.add_argument("--graph-all", action="store_true",
                    help="also replay the step as a CUDA graph at N > 1 (device-side all-reduce epochs)")
    ap.add_argument("--double-backward", action="store_true",
                    help="force-training step (SURVEY §8(f) row 1): fwd + bwd + the double backward "
                         "(dB_bar, A_bar, W_bar of <uA, dA>) per step; metric symcon_fwd_bwd_bwd2_nodes_per_s")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
def shape_of(name):
    from synth.inputs import CONFIGS
    return CONFIGS[name]


def plan_bins(world, seed=0):
    """Alg. 1 over the Table-2 manifest (same plan on every rank: deterministic)."""
    from synth.inputs import table2_sizes
    from paper_2504_10700_b200 import _lib
    sizes = table2_sizes(seed=seed)
    t0 = time.time()
    offs, ids = _lib.symcon_pack_balanced(sizes, CAPACITY, world)
    return sizes, offs, ids, time.time() - t0


def bin_elements(sizes, offs, ids, b, n_elements):
    from synth.inputs import graph_elements
    g = ids[offs[b]:offs[b + 1]]
    return graph_elements(sizes[g], n_elements=n_elements, seed=0, salt=int(b))


def alg_ops(sc):
    """Algorithmic FP32 lane-ops per (node, channel), per kernel and for the whole path, counted
    from the plan's tables; each is the op count of the exact evaluation the
    kernel performs, which is the smallest we know (so the roofline stays a bound):
      fwd  = prefix products (a,b) + degree-3 monomials + folded rows   (monomials, then one FMA per row)
      dW   = same products + folded rows                                 (S_j += dB_o * mono_j)
      dA   = prefix products of degree-3 monomials + folded rows (g_j) + 2 per degree-3 monomial
             + 2 per prefix group + 1 per degree-1 monomial          (reverse of the prefix structure)
      path = fwd + dA + dW with the backward's products shared."""
    from paper_2504_10700_b200 import _lib
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
    fwd = products + n_fold
    dW = products + n_fold
    dA = len(prefixes3) + n_fold + 2 * deg3 + 2 * len(prefixes) + deg1
    path = fwd + (products + n_fold) + (n_fold + 2 * deg3 + 2 * len(prefixes) + deg1)
    # double backward (codegen symcon_bwd2 / symcon_bwd2_dW): per prefix p' (2 ops), p for degree-3
    # groups (1); per degree-3 monomial mono' (2) and, in the tile kernel, A_bar_c, h, h' (3); per
    # row one FMA into dB_bar (+ one into g for degree >= 2); per prefix group 2 (4 with h') FMAs
    # into A_bar_a, A_bar_b. W_bar: products as above + one FMA per row.
    rows1 = sum(1 for r in rows if deg[r[2]] == 1)
    p3 = len(prefixes3)
    bwd2 = rows1 + 2 * (n_fold - rows1) + 2 * len(prefixes) + p3 + 5 * deg3 + 4 * p3 + 2 * (len(prefixes) - p3)
    bwd2_dW = n_fold + 2 * len(prefixes) + p3 + 2 * deg3
    return {"fwd": fwd, "dA": dA, "dW": dW, "path": path, "bwd2": bwd2, "bwd2_dW": bwd2_dW, "n_fold": n_fold, "products": products,
            "prefixes": len(prefixes), "deg3_monomials": deg3, "n_sym": int(len(L))}


def path_roofline(cfg, sc, mean_nodes, path_ops, ms_step, dbl):
    """Whole-step roofline: the step's algorithmic FP32 lane-ops at the ALU peak vs its
    algorithmic HBM bytes at the measured copy bandwidth (A read twice, dB, B and dA
    once per node-channel; the double backward adds uA, A, dB reads and dB_bar, A_bar writes)."""
    K = cfg.channels
    nlm = (cfg.lmax_in + 1) ** 2
    outc = sc.out_dim // K
    per = 4 * (2 * nlm + outc + outc + nlm)
    if dbl:
        per += 4 * (3 * nlm + outc + outc + nlm)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    t_alu = path_ops / (148 * 128 * 1.965e9)
    t_hbm = per * mean_nodes * K / (hbm * 1e9)
    bound = "alu" if t_alu >= t_hbm else "hbm"
    return {"bound": bound, "frac": max(t_alu, t_hbm) / (ms_step / 1e3), "t_alu_ms": t_alu * 1e3, "t_hbm_ms": t_hbm * 1e3,
            "bytes_per_node_channel": per}


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
def cpu_baseline(cfg, sc, A, W, ne, dB, n_sample, seed=0):
    """The oracle's plain C fp64 loop (never tuned) on a bounded sample of the workload."""
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
    return {"value": len(idx) / dt, "unit": "nodes/s", "cores": oc.threads(), "kind": "oracle",
            "sample": f"{len(idx)} random nodes of one {A.shape[0]}-node bin, fwd+bwd (B, dA, dW), fp64 C/OpenMP loop "
                      f"over {oc.n_terms} raw U terms per (node, channel), {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle on the host cores, each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from synth.inputs import gen_A, gen_W, gen_dB
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    cfg = shape_of(args.config)
    prob = Problem(cfg.lmax_in, cfg.correlation, cfg.out_L)
    oc = OracleC(prob)
    sizes, offs, ids, _ = plan_bins(max(args.gpus, 1))
    ne_full = bin_elements(sizes, offs, ids, 0, cfg.n_elements)
    n_bin = len(ne_full)
    per_step = max(64, args.cpu_sample // 8)
    A = gen_A(per_step, cfg.channels, 16, "cpu").numpy()
    W = gen_W(cfg.n_elements, prob.block_sizes(), cfg.channels, "cpu").numpy()
    dB = gen_dB(per_step, prob.out_dim(cfg.channels), "cpu").numpy()
    ne = ne_full[:per_step]
    for _ in range(args.warmup):
        oc.forward(A[:16], W, ne[:16])
    t0 = time.time()
    for _ in range(args.steps):
        oc.forward(A, W, ne)
        oc.backward(A, W, ne, dB)
    dt = time.time() - t0
    v = per_step * args.steps / dt
    out = {"impl": "reference", "metric": "symcon_fwd_bwd_nodes_per_s", "value": v, "unit": "nodes/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config}_dp_step", "nodes_per_bin": n_bin, "channels": cfg.channels,
                      "out": "+".join(f"{L}{'e' if L % 2 == 0 else 'o'}" for L in cfg.out_L), "lmax_in": cfg.lmax_in,
                      "correlation": cfg.correlation, "elements": cfg.n_elements,
                      "sample": f"{per_step} nodes of bin 0 per step"},
           "cpu_baseline": {"value": v, "unit": "nodes/s", "cores": oc.threads(), "kind": "oracle",
                            "sample": f"{per_step} nodes per step x {args.steps} steps"},
           "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


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
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200 import _lib
    from synth.inputs import gen_A, gen_W, gen_dB
    cfg = shape_of(args.config)
    sc = SymmetricContraction(cfg.lmax_in, cfg.correlation, cfg.out_L, cfg.n_elements, cfg.channels, device=local)

    from paper_2504_10700_b200.dist import BinPackedShards, DataParallelContraction
    from synth.inputs import table2_sizes
    sizes = table2_sizes(seed=0)
    t0 = time.time()
    shards = BinPackedShards(sizes, CAPACITY, world, rank)
    t_pack = time.time() - t0
    n_bins = shards.n_bins
    # pool of distinct bins for this rank (cycled): steps 0..POOL-1 of the epoch
    pool = []
    uA = {}
    for q in range(POOL):
        step_id = q % shards.n_steps
        b = shards.bin_of(step_id)
        ne = torch.from_numpy(bin_elements(sizes, shards.offsets, shards.ids, b, cfg.n_elements)).to(dev)
        N = ne.numel()
        A = gen_A(N, cfg.channels, sc.n_lm, dev, seed=100 * q + rank)
        dB = gen_dB(N, sc.out_dim, dev, seed=100 * q + rank)
        B = torch.empty((N, sc.out_dim), device=dev)
        dA = torch.empty_like(A)
        pool.append((b, N, A, ne, dB, B, dA))
        if args.double_backward:
            uA[q] = gen_A(N, cfg.channels, sc.n_lm, dev, seed=100 * q + rank + 7)
    imbalance = max(shards.step_imbalance(q % shards.n_steps) for q in range(POOL))
    W = gen_W(cfg.n_elements, sc.block_sizes(), cfg.channels, dev)
    if world > 1:
        dist.broadcast(W, 0)
    dW = torch.empty_like(W)
    for q in range(POOL):
        sc.workspace(pool[q][1])
    conc = False if args.sequential_bwd else (True if args.concurrent_bwd else None)
    dp = DataParallelContraction(sc, overlap=not args.no_overlap, concurrent_bwd=conc, allreduce=args.allreduce)

    def bwd2(q, A, ne, dB, runner):
        # double backward of the same step (force loss): uA terms through symcon_backward2, W_bar
        # all-reduced over ranks like dW
        runner.backward2(A, W, ne, dB, uA[q % POOL])

    def step(q):
        b, N, A, ne, dB, B, dA = pool[q % POOL]
        dp.forward(A, W, ne, B=B)
        dp.backward(A, W, ne, dB, dA=dA, dW=dW)
        if args.double_backward:
            bwd2(q, A, ne, dB, dp)
        return N

    for q in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    assert s == 0, (s, bad)
    use_graph = (world == 1 or args.graph_all) and not args.no_graph
    if use_graph:
        # one CUDA graph per pool entry (the whole step: bucketing, fold, fwd, dW || dA, reduce,
        # unfold); replays remove the per-launch gaps. Launch counts are taken at capture.
        graphs, per_step = [], []
        for q in range(POOL):
            g = torch.cuda.CUDAGraph()
            n0 = dp.launches
            with torch.cuda.graph(g):
                step(q)
            per_step.append(dp.launches - n0)
            graphs.append(g)
        torch.cuda.synchronize()
        eager_step = step

        def step(q):  # noqa: F811
            graphs[q % POOL].replay()
            dp.launches += per_step[q % POOL]
            if getattr(dp, "_peer", None) is not None:
                # graph q was captured with buffer parity q % 2; keep eager calls alternating too
                dp._peer.parity = (q + 1) % 2
            return pool[q % POOL][1]
        for q in range(POOL):   # a whole cycle, so the timed replays continue the buffer alternation
            step(q)
        torch.cuda.synchronize()
    if getattr(dp, "_peer", None) is not None:
        assert int(dp._peer.err.item()) == 0, "peer all-reduce barrier timed out"
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.symcon_profile_reset(sc.plan)
    dp.launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nodes = 0
    with ClockSampler(local) as clk:
        # ranks enter the timed region together (the sampler start-up takes a variable fraction
        # of a second per rank; without this barrier the first rank's wait is charged to the others)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.start()
        e0.record()
        for q in range(args.steps):
            nodes += step(q)
        e1.record()
        torch.cuda.synchronize()
        clk.end()
    if world > 1:
        dist.barrier()
    if getattr(dp, "_peer", None) is not None:
        assert int(dp._peer.err.item()) == 0, "peer all-reduce barrier timed out"
    ms = e0.elapsed_time(e1)
    # per-kernel times for the roofline: a separate pass with the kernels back to back on one
    # stream (the throughput region above overlaps dW and dA, which would blur each kernel's time)
    _lib.symcon_profile_enable(sc.plan, 1)
    _lib.symcon_profile_reset(sc.plan)
    seq = DataParallelContraction(sc, overlap=not args.no_overlap, concurrent_bwd=False, allreduce="nccl")
    launches_timed = dp.launches
    for q in range(args.steps):
        b_, N_, A_, ne_, dB_, B_, dA_ = pool[q % POOL]
        seq.forward(A_, W, ne_, B=B_)
        seq.backward(A_, W, ne_, dB_, dA=dA_, dW=dW)
        if args.double_backward:
            bwd2(q, A_, ne_, dB_, seq)
    torch.cuda.synchronize()
    prof = _lib.symcon_profile_read(sc.plan)
    _lib.symcon_profile_enable(sc.plan, 0)
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
    hU = uA[0].cpu().pin_memory() if args.double_backward else None
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
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    t2 = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = N * world / (float(t2[0]) / 1e3)
    h2d = hA.numel() * 4 + hne.numel() * 4 + hdB.numel() * 4 + (hU.numel() * 4 if hU is not None else 0)
    d2h = hdW.numel() * 4 * (2 if args.double_backward else 1)

    if rank == 0:
        ops = alg_ops(sc)
        K = cfg.channels
        clocks = clk.summary()
        # dominant kernel by measured time
        kern = max(prof, key=lambda k: prof[k][1]) if prof else None
        roof = None
        if kern:
            cnt, tot_ms = prof[kern]
            avg_ms = tot_ms / max(cnt, 1)
            per_nc = {"symcon_fwd": ops["fwd"], "symcon_bwd_dA": ops["dA"], "symcon_bwd_dW": ops["dW"],
                      "symcon_bwd2": ops["bwd2"], "symcon_bwd2_dW": ops["bwd2_dW"]}.get(kern)
            mean_nodes = nodes / args.steps
            if per_nc:
                achieved = per_nc * mean_nodes * K / (avg_ms / 1e3) / 1e12  # T lane-ops/s
                sm_mhz = 1965.0
                peak = 148 * 128 * sm_mhz * 1e6 / 1e12
                nlm = (cfg.lmax_in + 1) ** 2
                outc = sc.out_dim // K
                alg_b = {"symcon_fwd": 4 * (nlm + outc), "symcon_bwd_dA": 4 * (2 * nlm + outc),
                         "symcon_bwd_dW": 4 * (nlm + outc), "symcon_bwd2": 4 * (4 * nlm + 2 * outc),
                         "symcon_bwd2_dW": 4 * (2 * nlm + outc)}[kern] * mean_nodes * K
                traffic, tsrc = None, None
                tpath = os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")
                if os.path.exists(tpath) and args.config == "mp_medium":
                    tj = json.load(open(tpath))
                    rec = tj["kernels"].get(kern)
                    if rec:
                        traffic = rec["dram_bytes_read"] + rec["dram_bytes_write"]
                        tsrc = tj["source"]
                # the binding resource: ALU time at the FP32 peak vs HBM time at the measured copy
                # bandwidth, both from the kernel's algorithmic work
                hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
                    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
                t_alu = per_nc * mean_nodes * K / (peak * 1e12)
                t_hbm = alg_b / (hbm_peak * 1e9)
                if t_hbm > t_alu:
                    gbs = alg_b / (avg_ms / 1e3) / 1e9
                    roof = {"bound": "hbm", "kernel": kern, "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                            "frac": gbs / hbm_peak, "traffic": traffic, "traffic_source": tsrc,
                            "algorithmic_bytes": alg_b, "avg_launch_ms": avg_ms, "ops_per_node_channel": per_nc,
                            "alu_tops": achieved, "alu_frac": achieved / peak,
                            "peak_derivation": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
                else:
                    roof = {"bound": "alu", "kernel": kern, "achieved": achieved, "peak": peak,
                            "unit": "Tops/s (fp32 FMA lane-ops)",
                            "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                            "algorithmic_bytes": alg_b, "avg_launch_ms": avg_ms,
                            "ops_per_node_channel": per_nc, "hbm_gbs": alg_b / (avg_ms / 1e3) / 1e9,
                            "peak_derivation": "148 SMs x 128 FP32 lanes x 1965 MHz (clocks.max.sm); FFMA probe measured 36.0 T/s"}
        path_ops = (ops["path"] + (ops["bwd2"] + ops["bwd2_dW"] if args.double_backward else 0)) * (nodes / args.steps) * K
        kernels = {k: {"launches": v[0], "avg_ms": v[1] / max(v[0], 1)} for k, v in prof.items()}
        out = {
            "metric": "symcon_fwd_bwd_bwd2_nodes_per_s" if args.double_backward else "symcon_fwd_bwd_nodes_per_s", "value": value, "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}_dp_step" + ("_double_backward" if args.double_backward else ""), "model": "MACE symmetric contraction",
                       "channels": K, "out": "+".join(f"{K}x{L}{'e' if L % 2 == 0 else 'o'}" for L in cfg.out_L),
                       "lmax_in": cfg.lmax_in, "correlation": cfg.correlation, "elements": cfg.n_elements,
                       "capacity_nodes": CAPACITY, "bins": n_bins, "global_batch": int(nodes_all / args.steps),
                       "step_imbalance_max_over_mean": round(imbalance, 5), "dW_allreduce": ({"peer": "libsymcon NVLink peer-memory kernel (symmetric buffers), dA concurrent",
                                                        "nccl": "NCCL on a communication stream"}[dp.allreduce]
                                                       if world > 1 else None),
                       "seq_len": None, "parallelism": f"dp{world}", "l2": "inputs > L2 (A 410 MB/bin), 4-bin pool",
                       "alg1_pack_s": round(t_pack, 3), "cuda_graph": use_graph},
            "per_gpu_nodes_per_s": value / world,
            "per_rank_ms_per_step": per_rank_ms,
            "path_tops": path_ops / (ms_max / args.steps / 1e3) / 1e12,
            "path_frac_of_alu_peak": path_ops / (ms_max / args.steps / 1e3) / 1e12 / (148 * 128 * 1.965e-3),
            "path_roofline": path_roofline(cfg, sc, nodes / args.steps, path_ops, ms_max / args.steps, args.double_backward),
            "roofline": roof, "kernels": kernels, "alg_ops_per_node_channel": ops,
            "clocks": clocks, "gpu_launches": launches_timed,
            "kernel_timing": "per-kernel CUDA events from a separate pass of the same steps with dW and dA back to back",
            "e2e": {"value": e2e_value, "unit": "nodes/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "note": "H2D A+node_elem+dB from pinned host, D2H dW, per step through SymmetricContraction; "
                            "the copy of step s+1 (copy stream) overlaps the compute of step s"},
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, sc, A, W, ne, dB, args.cpu_sample)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


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
                                x["dh"].data_ptr(), x["dR"].data_ptr(), ws.data_ptr(), ws.numel(), st)
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
                                     dev_bufs["dA"])
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

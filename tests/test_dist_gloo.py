"""Multi-process (gloo, world_size 2, CPU) checks of the data-parallel plumbing.

The CUDA kernels need a GPU, so the per-rank dW here comes from the oracle's C evaluator on
the rank's bin; what is tested is the sharding (Alg. 1 bins -> ranks -> steps, every graph
exactly once) and that the SUM all-reduce of per-rank dW equals dW over the union of bins.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _graph_inputs(gids, sizes, K, P, E, seed=0):
    """Per-graph seeded A, dB, node elements (identical on every rank for the same graph)."""
    A, dB, ne = [], [], []
    for g in gids:
        rng = np.random.default_rng([seed, int(g)])
        n = int(sizes[g])
        A.append(rng.normal(size=(n, K, 16)).astype(np.float32))
        dB.append(rng.normal(size=(n, K)).astype(np.float32))
        ne.append(rng.integers(0, E, size=n).astype(np.int32))
    if not A:
        return np.zeros((0, K, 16), np.float32), np.zeros((0, K), np.float32), np.zeros(0, np.int32)
    return np.concatenate(A), np.concatenate(dB), np.concatenate(ne)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_10700_b200.dist import BinPackedShards
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    rng = np.random.default_rng(5)
    sizes = rng.integers(1, 40, size=120)
    C, K, E = 100, 4, 3
    prob = Problem(3, 3, (0,))
    oc = OracleC(prob)
    W = np.random.default_rng(2).normal(size=(E, prob.n_paths, K)).astype(np.float32)
    sh = BinPackedShards(sizes, C, world, rank)
    mine = []
    for step in range(sh.n_steps):
        gids = sh.graphs(step)
        mine.extend(int(g) for g in gids)
        A, dB, ne = _graph_inputs(gids, sizes, K, prob.n_paths, E)
        _, dW = oc.backward(A, W, ne, dB, want_dA=False) if len(ne) else (None, np.zeros(W.shape))
        # double backward (force loss): W_bar is a W gradient too and is all-reduced the same way
        uA = np.cos(A) if len(ne) else A
        Wb = oc.backward2(A, W, ne, dB, uA, want_dB=False, want_A=False)[2] if len(ne) else np.zeros(W.shape)
        t = torch.from_numpy(dW.astype(np.float64))
        tb = torch.from_numpy(Wb.astype(np.float64))
        dist.all_reduce(t)                                   # SUM over ranks (the NCCL call on GPU)
        dist.all_reduce(tb)
        if rank == 0:
            gall = np.concatenate([sh.graphs(step, r) for r in range(world)])
            A2, dB2, ne2 = _graph_inputs(gall, sizes, K, prob.n_paths, E)
            _, ref = oc.backward(A2, W, ne2, dB2, want_dA=False)
            out.put(("step", step, float(np.abs(t.numpy() - ref).max()), float(np.abs(ref).max())))
            refb = oc.backward2(A2, W, ne2, dB2, np.cos(A2), want_dB=False, want_A=False)[2]
            out.put(("step", step, float(np.abs(tb.numpy() - refb).max()), float(np.abs(refb).max())))
    lst = [None] * world
    dist.all_gather_object(lst, mine)
    if rank == 0:
        allg = sorted(g for l in lst for g in l)
        out.put(("cover", allg == list(range(len(sizes))), sh.n_bins, float(sh.bin_loads().max())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_dw_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    steps = [m for m in msgs if m[0] == "step"]
    cover = [m for m in msgs if m[0] == "cover"]
    assert steps and cover
    for _, s, err, scale in steps:
        assert err <= 1e-12 * max(scale, 1.0), (s, err)
    ok, n_bins, max_load = cover[0][1:]
    assert ok and n_bins % 2 == 0 and max_load <= 100


def test_bin_packed_shards_single_process():
    from paper_2504_10700_b200.dist import BinPackedShards
    from synth.inputs import table2_sizes
    sizes = table2_sizes(scale=0.02)
    for world in (1, 2, 4, 8):
        sh = BinPackedShards(sizes, 50_000, world, 0)
        assert sh.n_bins % world == 0
        seen = np.zeros(len(sizes), np.int32)
        for s in range(sh.n_steps):
            for r in range(world):
                seen[sh.graphs(s, r)] += 1
        assert (seen == 1).all()
        assert sh.bin_loads().max() <= 50_000
        if sh.n_steps > 1:
            assert sh.step_imbalance(0) < 1.02    # bins of the first round are filled to C - 768

"""Partition-quality study: Alg. 1 (libsymcon's C++
partitioner) against the usual alternatives on the synthetic Table-2 epoch, with the paper's
Eq. (1)-(3) metrics and the per-step GPU balance that drives data-parallel
step time; node key (reading s19) and an edge-aware key.

    python tools/partition_study.py [--scale 0.1] [--capacity 50000] [--gpus 8] [--out profiles/r01/partition_study.json]

Baselines (host analysis code, not part of the product path):
  fixed-count  shuffled graphs, a fixed number of graphs per batch (PyTorch's default batching),
               chosen so the mean batch holds C nodes; bins may exceed C.
  FFD / BFD    first-fit / best-fit decreasing with capacity C (GareyJohnson1979 in the paper).
Bins go to GPUs round-robin (bin j -> GPU j % G, step j // G) for every method, as for Alg. 1.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def edges_of(sizes, deg=30):
    """Edge count of each graph under the synthetic TP graph recipe (synth.inputs.gen_tp_graph)."""
    sizes = np.asarray(sizes, dtype=np.int64)
    return sizes * np.minimum(deg, np.maximum(sizes - 1, 0))


def pack_alg1(sizes, C, G):
    from paper_2504_10700_b200 import _lib
    offs, ids = _lib.symcon_pack_balanced(np.asarray(sizes, dtype=np.int64), C, G)
    return [ids[offs[b]:offs[b + 1]] for b in range(len(offs) - 1)]


def pack_fixed_count(sizes, C, seed=0):
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(sizes))
    per = max(1, int(round(C / float(np.mean(sizes)))))
    return [order[i:i + per] for i in range(0, len(order), per)]


class _MaxTree:
    """Segment tree of the bins' remaining capacities; leftmost bin with remaining >= s."""

    def __init__(self, n, C):
        self.n = 1
        while self.n < n:
            self.n *= 2
        self.t = np.full(2 * self.n, -1, dtype=np.int64)
        self.C = C

    def set(self, i, v):
        i += self.n
        self.t[i] = v
        i //= 2
        while i:
            self.t[i] = max(self.t[2 * i], self.t[2 * i + 1])
            i //= 2

    def leftmost(self, s):
        if self.t[1] < s:
            return -1
        i = 1
        while i < self.n:
            i = 2 * i if self.t[2 * i] >= s else 2 * i + 1
        return i - self.n


def pack_ffd(sizes, C):
    order = np.argsort(-np.asarray(sizes), kind="stable")
    tree = _MaxTree(len(sizes), C)
    bins, rem = [], []
    for g in order:
        s = int(sizes[g])
        b = tree.leftmost(s)
        if b < 0:
            b = len(bins)
            bins.append([])
            rem.append(C)
        bins[b].append(int(g))
        rem[b] -= s
        tree.set(b, rem[b])
    return [np.array(b, dtype=np.int64) for b in bins]


def pack_bfd(sizes, C):
    from sortedcontainers import SortedList
    order = np.argsort(-np.asarray(sizes), kind="stable")
    sl = SortedList()          # (remaining, bin id)
    bins = []
    for g in order:
        s = int(sizes[g])
        k = sl.bisect_left((s, -1))
        if k == len(sl):
            b, r = len(bins), C
            bins.append([])
        else:
            r, b = sl.pop(k)
        bins[b].append(int(g))
        sl.add((r - s, b))
    return [np.array(b, dtype=np.int64) for b in bins]


def metrics(bins, sizes, edges, C, G):
    sizes = np.asarray(sizes, dtype=np.int64)
    loads = np.array([sizes[b].sum() for b in bins], dtype=np.float64)
    eloads = np.array([edges[b].sum() for b in bins], dtype=np.float64)
    sq = np.array([(sizes[b].astype(np.float64) ** 2).sum() for b in bins])
    n_bins = len(bins)
    pad = n_bins + (-n_bins) % G                      # bins padded to full steps
    L = np.concatenate([loads, np.zeros(pad - n_bins)]).reshape(-1, G)
    EL = np.concatenate([eloads, np.zeros(pad - n_bins)]).reshape(-1, G)
    step_max, step_mean = L.max(1), L.mean(1)
    estep_max, estep_mean = EL.max(1), EL.mean(1)
    return {
        "bins_eq1": n_bins,
        "padding_eq2": float(sq.sum() / float(C) ** 2),
        "max_gap_eq3": float(sq.max() - sq.min()),
        "over_capacity_bins": int((loads > C).sum()),
        "fill_mean": float(loads.mean() / C),
        "steps": int(L.shape[0]),
        # data-parallel step time ~ the slowest GPU: sum over steps of max load vs ideal mean
        "dp_efficiency_nodes": float(step_mean.sum() / step_max.sum()),
        "dp_efficiency_edges": float(estep_mean.sum() / estep_max.sum()),
        "step_imbalance_nodes_p50": float(np.median(step_max / np.maximum(step_mean, 1))),
        "step_imbalance_nodes_max": float((step_max / np.maximum(step_mean, 1)).max()),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--capacity", type=int, default=50_000)
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "partition_study.json"))
    args = ap.parse_args()
    from synth.inputs import table2_sizes
    sizes = table2_sizes(seed=0, scale=args.scale)
    edges = edges_of(sizes)
    C, G = args.capacity, args.gpus
    res = {"graphs": int(len(sizes)), "nodes": int(sizes.sum()), "edges": int(edges.sum()), "capacity": C, "gpus": G,
           "scale": args.scale, "methods": {}}
    runs = [("alg1_node_key", lambda: pack_alg1(sizes, C, G)),
            ("alg1_edge_key", lambda: pack_alg1(edges, int(C * edges.sum() / sizes.sum()), G)),
            ("fixed_count", lambda: pack_fixed_count(sizes, C)),
            ("ffd", lambda: pack_ffd(sizes, C)),
            ("bfd", lambda: pack_bfd(sizes, C))]
    for name, fn in runs:
        t0 = time.time()
        bins = fn()
        dt = time.time() - t0
        m = metrics(bins, sizes, edges, C, G)
        m["pack_seconds"] = round(dt, 3)
        res["methods"][name] = m
        print(name, json.dumps(m), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Seeded input generators (SURVEY.md §8(d) "Synthetic inputs").

Seeds: A=1, W=2, node_elem=3, dB=4, graph sizes=5 (each offset by `seed`).
A, W and dB are drawn by a CPU torch generator and then moved to the requested
device, so a seed gives the same values on every device: the GPU arm of bench.py
and the oracle (reference arm, parity tests) see identical inputs. The TP inputs
(several GB per bin) are drawn on the requested device.
"""
from dataclasses import dataclass
import math

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    n_nodes: int
    channels: int
    n_elements: int
    out_L: tuple
    lmax_in: int = 3
    correlation: int = 3
    elem_dist: str = "uniform"     # uniform | organic | zipf
    graphs: str = "single"         # single | molecules


CONFIGS = {
    # BASELINE.json configs[0..3]
    "tiny": Config("tiny", 32, 16, 3, (0,), elem_dist="uniform"),
    "off_small": Config("off_small", 20_000, 96, 10, (0,), elem_dist="organic", graphs="molecules"),
    "mp_medium": Config("mp_medium", 50_000, 128, 89, (0, 1), elem_dist="zipf"),
    "large": Config("large", 200_000, 256, 89, (0, 1, 2), elem_dist="zipf"),
}

# Table 2: source, number of graphs, vertex range (inclusive)
TABLE2 = [
    ("Al-HCl(aq)", 884, 281, 281),
    ("CuNi", 74_335, 492, 500),
    ("HEA", 25_628, 36, 48),
    ("Liquid water", 190_267, 768, 768),
    ("MPtrj", 1_580_312, 1, 444),
    ("TMD", 219_627, 16, 96),
    ("Water clusters", 460_000, 9, 75),
    ("Zeolite", 99_770, 203, 408),
]
TABLE2_TOTAL = 2_650_823

ORGANIC = {"H": 0.45, "C": 0.33, "O": 0.09, "N": 0.07}   # rest 0.06 split evenly (unpinned)


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def zipf_probs(n, s=1.1):
    r = np.arange(1, n + 1, dtype=np.float64)
    p = r ** (-s)
    return p / p.sum()


def organic_probs(n):
    p = np.array(list(ORGANIC.values()) + [0.0] * max(0, n - len(ORGANIC)), dtype=np.float64)[:n]
    if n > len(ORGANIC):
        p[len(ORGANIC):] = (1.0 - sum(ORGANIC.values())) / (n - len(ORGANIC))
    return p / p.sum()


def elem_probs(cfg_or_dist, n):
    dist = cfg_or_dist.elem_dist if isinstance(cfg_or_dist, Config) else cfg_or_dist
    if dist == "zipf":
        return zipf_probs(n)
    if dist == "organic":
        return organic_probs(n)
    return np.full(n, 1.0 / n)


def gen_node_elem(n_nodes, n_elements, dist="uniform", device="cpu", seed=0):
    p = torch.tensor(elem_probs(dist, n_elements), dtype=torch.float64)
    if n_nodes == 0:
        return torch.zeros(0, dtype=torch.int32, device=device)
    g = _gen("cpu", 3 + seed)
    idx = torch.multinomial(p, n_nodes, replacement=True, generator=g)
    return idx.to(torch.int32).to(device)


def gen_A(n_nodes, channels, n_lm=16, device="cpu", seed=0):
    g = _gen("cpu", 1 + seed)
    return torch.randn((n_nodes, channels, n_lm), generator=g, dtype=torch.float32).to(device)


def gen_W(n_elements, block_sizes, channels, device="cpu", seed=0):
    """W [E][P][K] ~ N(0,1)/n_eta per (L, nu) block (MACE-style init; unpinned).

    block_sizes: [(L, nu, n_eta)] in W column order (the caller supplies it)."""
    g = _gen("cpu", 2 + seed)
    P = sum(b[2] for b in block_sizes)
    W = torch.randn((n_elements, P, channels), generator=g, dtype=torch.float32)
    scale = torch.cat([torch.full((b[2],), 1.0 / b[2]) for b in block_sizes])
    return (W * scale.view(1, P, 1)).to(device)


def gen_dB(n_nodes, out_dim, device="cpu", seed=0):
    g = _gen("cpu", 4 + seed)
    return torch.randn((n_nodes, out_dim), generator=g, dtype=torch.float32).to(device)


def graph_edges(sizes, deg=30):
    """Edges of graphs of the given vertex counts under the synthetic degree min(deg, n-1) per node
     -- the secondary load key of the DP step."""
    sizes = np.asarray(sizes, dtype=np.int64)
    return sizes * np.minimum(deg, np.maximum(sizes - 1, 0))


def molecule_sizes(total, lo=10, hi=100, seed=0):
    """OFF-small batch: molecules of U[lo, hi] atoms until the sum reaches `total` (last truncated)."""
    rng = np.random.default_rng(5 + seed)
    sizes = []
    s = 0
    while s < total:
        n = int(rng.integers(lo, hi + 1))
        n = min(n, total - s)
        sizes.append(n)
        s += n
    return sizes


def table2_sizes(seed=0, scale=1.0):
    """Graph vertex counts with Table 2's per-source counts (uniform within each range).

    scale < 1 keeps floor(count*scale) graphs per source (for small tests)."""
    rng = np.random.default_rng(5 + seed)
    parts = []
    for _, count, lo, hi in TABLE2:
        c = int(math.floor(count * scale)) if scale != 1.0 else count
        parts.append(rng.integers(lo, hi + 1, size=c, dtype=np.int64))
    return np.concatenate(parts)


def graph_elements(sizes, n_elements=89, seed=0, salt=0):
    """Per-node elements for a list of graphs: each graph draws 1-4 distinct elements
    (Zipf(1.1) over n_elements), then each node picks one of them uniformly (unpinned)."""
    rng = np.random.default_rng([5 + seed, 1 + salt])
    p = zipf_probs(n_elements)
    out = np.empty(int(np.sum(sizes)), dtype=np.int32)
    pos = 0
    for n in sizes:
        k = int(rng.integers(1, 5))
        els = rng.choice(n_elements, size=min(k, n_elements), replace=False, p=p)
        out[pos:pos + n] = els[rng.integers(0, len(els), size=n)]
        pos += n
    return out


def make_config_inputs(cfg, block_sizes, out_dim, device="cpu", seed=0, n_nodes=None):
    """(A, W, node_elem, dB) for one of CONFIGS (n_nodes overrides the batch size)."""
    N = cfg.n_nodes if n_nodes is None else n_nodes
    A = gen_A(N, cfg.channels, (cfg.lmax_in + 1) ** 2, device, seed)
    W = gen_W(cfg.n_elements, block_sizes, cfg.channels, device, seed)
    ne = gen_node_elem(N, cfg.n_elements, cfg.elem_dist, device, seed)
    dB = gen_dB(N, out_dim, device, seed)
    return A, W, ne, dB


# ------------------------------------------------------------------ channelwise TP (§8(f) row 2)
# Seeds: Y=6, h=7, R=8, graph=9 (each offset by `seed`). Degree: 30 incoming edges per node
# (deg ~45.6 for liquid water, others unpinned -> 30), capped at n-1 inside
# each molecule; senders uniform over the other nodes of the receiver's molecule.
def gen_tp_graph(sizes, deg=30, seed=0):
    """Receiver-sorted edge list (sender, receiver) int32 over molecules of the given sizes
    laid out consecutively."""
    rng = np.random.default_rng(9 + seed)
    sizes = np.asarray(sizes, dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    node_mol_start = np.repeat(starts, sizes)
    node_mol_size = np.repeat(sizes, sizes)
    N = int(sizes.sum())
    d = np.minimum(deg, node_mol_size - 1)
    receiver = np.repeat(np.arange(N, dtype=np.int64), d)
    # sender = another node of the same molecule: offset in [1, n-1] from the receiver, cyclic
    n = np.repeat(node_mol_size, d)
    off = 1 + (rng.random(receiver.shape[0]) * (n - 1)).astype(np.int64)
    local = (receiver - np.repeat(node_mol_start, d) + off) % n
    sender = np.repeat(node_mol_start, d) + local
    return sender.astype(np.int32), receiver.astype(np.int32)


def gen_tp_inputs(n_nodes, n_edges, channels, n_y, n_h, n_paths, device="cpu", seed=0):
    gy, gh, gr = _gen(device, 6 + seed), _gen(device, 7 + seed), _gen(device, 8 + seed)
    Y = torch.randn((n_edges, n_y), generator=gy, device=device, dtype=torch.float32)
    h = torch.randn((n_nodes, n_h, channels), generator=gh, device=device, dtype=torch.float32)
    R = torch.randn((n_edges, n_paths, channels), generator=gr, device=device, dtype=torch.float32)
    return Y, h, R

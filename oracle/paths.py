"""Coupling paths and generalized CG tensors U (oracle; test infrastructure only).

PAPER.md:558-588 (Alg. 3) sums, for each output (L, M) and correlation order
nu = 1..nu_max, over "all combinations lm of l1m1, ..., l_nu m_nu" weighted by
the generalized Clebsch-Gordan coefficient C^{LM}_{lm} (symbol only,
PAPER.md:306, 562). Reading s4: C^{LM}_{lm} is a left-nested
chain of pairwise real couplings (l1 (x) l2 -> L2, L2 (x) l3 -> L3, ...), every
intermediate allowed for nu <= 3, last intermediate = L; a path is kept iff
sum(l) + L is even (natural parity, reading s9). One weight per path eta
(reading s5): W[z, (L, nu, eta), k].

Reading s4b (nu = 4, correlation 4; SURVEY.md §8(c) s4 "corr-4 mid-filter"): the intermediates of a
nu = 4 chain are restricted to natural-parity irreps, L_j + l_1 + ... + l_j even at every coupling
step, L_j < 12 (MACE's filter_ir_mid for correlation 4). The paper's "all possible combinations ...
that would result in a nonzero contribution" holds: the filter keeps the complete
invariant space, pinned by the symmetrized rank = the multiplicity of L in Sym^4(0e+1o+2e+3o)
(23, 31, 46 for L = 0, 1, 2; tests/test_oracle_paths.py) with 158 / 284 / 358 of the 204 / 520 / 720
unfiltered chains.

eta order inside (L, nu): lexicographic on the interleaved key
(l1, l2, L2, l3, L3, ...).
"""
from dataclasses import dataclass, field
from itertools import product

import numpy as np

from .so3 import real_cg, lm_index

NONZERO_U = 1e-13


@dataclass
class Path:
    L: int
    nu: int
    ls: tuple          # (l1..l_nu)
    mids: tuple        # intermediates (L2..L_nu); for nu=1 empty; last == L for nu>=2
    eta: int = -1
    col: int = -1      # column in W's middle axis
    # raw ordered-tuple nonzeros: list of (M, (t1..t_nu), value), t_j in [0, (lmax+1)^2)
    terms: list = field(default_factory=list)


def _tri(a, b):
    return range(abs(a - b), a + b + 1)


def enumerate_paths(lmax_in, nu, L):
    """All left-nested paths of order nu ending in L (sorted by interleaved key)."""
    found = []
    for ls in product(range(lmax_in + 1), repeat=nu):
        if (sum(ls) + L) % 2:
            continue
        if nu == 1:
            if ls[0] == L:
                found.append(((ls[0],), ls, ()))
            continue
        # walk intermediates
        stack = [((ls[0],), ls[0], ())]
        for j in range(1, nu):
            nxt = []
            for key, cur, mids in stack:
                for Lj in _tri(cur, ls[j]):
                    if nu == 4 and ((Lj + sum(ls[:j + 1])) % 2 or Lj >= 12):
                        continue   # reading s4b: natural-parity intermediates at nu = 4
                    nxt.append((key + (ls[j], Lj), Lj, mids + (Lj,)))
            stack = nxt
        for key, cur, mids in stack:
            if cur == L:
                found.append((key, ls, mids))
    found.sort(key=lambda x: x[0])
    return [Path(L=L, nu=nu, ls=ls, mids=mids) for _, ls, mids in found]


def path_tensor(path):
    """Dense U[M, m1..m_nu] of one path (indices shifted by +l): chain of real CGs.

    T_1[M1, m1] = delta; T_j[Mj, m1..mj] = sum_{M_{j-1}} C^{Lj}_{L_{j-1} l_j}[Mj, M_{j-1}, m_j] T_{j-1}[...].
    """
    l1 = path.ls[0]
    T = np.eye(2 * l1 + 1)
    cur = l1
    for j in range(1, path.nu):
        lj, Lj = path.ls[j], path.mids[j - 1]
        C = real_cg(cur, lj, Lj)                    # [Lj][cur][lj]
        T = np.tensordot(C, T, axes=([1], [0]))      # [Lj][lj][m1..m_{j-1}]
        T = np.moveaxis(T, 1, -1)                    # [Lj][m1..m_{j-1}][lj]
        cur = Lj
    return T


def build_paths(lmax_in, correlation, out_L):
    """All paths for the output irreps, with W columns (L in out_L order, then nu, then eta)
    and raw ordered-tuple nonzeros."""
    paths = []
    col = 0
    for L in out_L:
        for nu in range(1, correlation + 1):
            for eta, p in enumerate(enumerate_paths(lmax_in, nu, L)):
                p.eta, p.col = eta, col
                col += 1
                U = path_tensor(p)
                for idx in zip(*np.nonzero(np.abs(U) > NONZERO_U)):
                    M = idx[0] - L
                    ts = tuple(lm_index(p.ls[j], idx[1 + j] - p.ls[j]) for j in range(p.nu))
                    p.terms.append((M, ts, float(U[idx])))
                paths.append(p)
    return paths


def eta_counts(lmax_in, correlation, L):
    return tuple(len(enumerate_paths(lmax_in, nu, L)) for nu in range(1, correlation + 1))


def dense_U(path, lmax_in):
    """U embedded in the full (lmax+1)^2 index space: [2L+1][n]*nu (brute force only)."""
    n = (lmax_in + 1) ** 2
    U = np.zeros((2 * path.L + 1,) + (n,) * path.nu)
    T = path_tensor(path)
    for idx in zip(*np.nonzero(T)):
        ts = tuple(lm_index(path.ls[j], idx[1 + j] - path.ls[j]) for j in range(path.nu))
        U[(idx[0],) + ts] = T[idx]
    return U

"""Pins for oracle/paths.py: counts, hand counts, representation-theory ranks, equivariance."""
import json
import os
from itertools import permutations, product

import numpy as np

from oracle.paths import build_paths, enumerate_paths, eta_counts, path_tensor
from oracle.so3 import real_cg, wigner_d_fit, random_rotation

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "derived_counts.json")))


def test_eta_counts():
    for L in (0, 1, 2):
        assert list(eta_counts(3, 3, L)) == GOLD["eta"][str(L)]


def test_hand_count_L0_nu3():
    # ordered (l1,l2,l3) with l1+l2+l3 even and (l1 (x) l2) containing l3 (the only L2 = l3
    # route to L=0): 1 + 3 + 3 + 3 + 3 + 6 + 1 + 3 = 23; brute-force here
    n = 0
    for l1, l2, l3 in product(range(4), repeat=3):
        if (l1 + l2 + l3) % 2 == 0 and abs(l1 - l2) <= l3 <= l1 + l2:
            n += 1
    assert n == 23 == len(enumerate_paths(3, 3, 0))


def test_raw_nnz():
    for L in (0, 1, 2):
        ps = build_paths(3, 3, [L])
        got = [sum(len(p.terms) for p in ps if p.nu == nu) for nu in (1, 2, 3)]
        assert got == GOLD["raw_nnz"][str(L)]


def test_nu1_identity_and_nu2_is_cg():
    for L in range(4):
        (p,) = enumerate_paths(3, 1, L)
        assert np.array_equal(path_tensor(p), np.eye(2 * L + 1))
    for p in enumerate_paths(3, 2, 1):
        assert np.array_equal(path_tensor(p), real_cg(p.ls[0], p.ls[1], 1))


def test_eta_order_lexicographic_interleaved():
    ps = enumerate_paths(3, 3, 1)
    keys = [(p.ls[0], p.ls[1], p.mids[0], p.ls[2], p.mids[1]) for p in ps]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


def _haar(f, n=4000):
    th = (np.arange(n) + 0.5) * np.pi / n
    return np.sum(f(th) * (1 - np.cos(th)) / np.pi) * np.pi / n


def _chi(l, th):
    return np.sin((2 * l + 1) * th / 2) / np.sin(th / 2)


def _sym_multiplicity(nu, L, lmax=3):
    """Multiplicity of (L, parity (-1)^L) in Sym^nu(0e+1o+2e+3o) by O(3) character integration."""
    def chiV(th, improper):
        return sum(((-1) ** l if improper else 1) * _chi(l, th) for l in range(lmax + 1))

    def chiSym(th, improper):
        c1 = chiV(th, improper)
        c2 = chiV(2 * th, False)
        if nu == 1:
            return c1
        if nu == 2:
            return (c1 ** 2 + c2) / 2
        c3 = chiV(3 * th, improper)
        return (c1 ** 3 + 3 * c1 * c2 + 2 * c3) / 6

    p = (-1) ** L
    m = 0.5 * (_haar(lambda t: chiSym(t, False) * _chi(L, t)) + p * _haar(lambda t: chiSym(t, True) * _chi(L, t)))
    return int(round(m))


def _symmetrized_rank(L, nu):
    rows = []
    for p in [q for q in build_paths(3, 3, [L]) if q.nu == nu]:
        acc = {}
        for M, ts, u in p.terms:
            key = (M, tuple(sorted(ts)))
            acc[key] = acc.get(key, 0.0) + u
        rows.append(acc)
    keys = sorted(set(k for r in rows for k in r))
    mat = np.array([[r.get(k, 0.0) for k in keys] for r in rows])
    return np.linalg.matrix_rank(mat, tol=1e-9)


def test_symmetrized_rank_equals_character_multiplicity():
    for L in (0, 1, 2):
        mult = [_sym_multiplicity(nu, L) for nu in (1, 2, 3)]
        assert mult == GOLD["sym_rank"][str(L)]
        assert [_symmetrized_rank(L, nu) for nu in (1, 2, 3)] == mult


def test_path_tensor_equivariance():
    rng = np.random.default_rng(4)
    R = random_rotation(rng)
    D = {l: wigner_d_fit(l, R) for l in range(4)}
    for L in (0, 1, 2):
        for p in enumerate_paths(3, 3, L)[::5]:
            T = path_tensor(p)
            lhs = np.einsum("Mabc,ai,bj,ck->Mijk", T, D[p.ls[0]], D[p.ls[1]], D[p.ls[2]])
            rhs = np.einsum("MN,Nijk->Mijk", D[L], T)
            assert np.allclose(lhs, rhs, atol=1e-11)

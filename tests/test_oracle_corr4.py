"""Pins for the correlation-4 oracle (reading s4b in oracle/paths.py and
DESIGN.md §3): nu = 4 chains with natural-parity intermediates.

* completeness of the filtered path set: the rank of the symmetrized nu = 4 tables equals the
  multiplicity of L in Sym^4(0e+1o+2e+3o), computed independently by O(3) character integration
  (23, 31, 46 for L = 0, 1, 2), i.e. the filter loses no invariant ("all possible
  combinations ... that would result in a nonzero contribution");
* nu = 4 U tensors are equivariant (Wigner-D fitted from scipy SH samples, independent of the CG code);
* the forward equals the dense brute force over all 16^4 tuples; rotation equivariance and inversion
  parity of B; the homogeneity split isolates the nu = 4 order (degree-4 scaling);
* the backward equals central finite differences; Euler identity with nu up to 4;
* the C evaluator equals the Python oracle at correlation 4.
"""
import numpy as np
import pytest

from oracle.contraction import Problem, forward, backward, forward_bruteforce
from oracle.paths import enumerate_paths, path_tensor, build_paths
from oracle.so3 import block_diag_d, random_rotation, wigner_d_fit, lm_index


def _haar(f, n=4000):
    th = (np.arange(n) + 0.5) * np.pi / n
    return np.sum(f(th) * (1 - np.cos(th)) / np.pi) * np.pi / n


def _chi(l, th):
    return np.sin((2 * l + 1) * th / 2) / np.sin(th / 2)


def _sym4_multiplicity(L, lmax=3):
    """Multiplicity of (L, (-1)^L) in Sym^4(V), V = 0e+1o+..., by the cycle-index formula
    chi_Sym4(g) = (c1^4 + 6 c1^2 c2 + 3 c2^2 + 8 c1 c3 + 6 c4) / 24, c_k = chi_V(g^k)."""
    def chiV(th, improper):
        return sum(((-1) ** l if improper else 1) * _chi(l, th) for l in range(lmax + 1))

    def chiS(th, improper):
        c1, c2, c3, c4 = chiV(th, improper), chiV(2 * th, False), chiV(3 * th, improper), chiV(4 * th, False)
        return (c1 ** 4 + 6 * c1 ** 2 * c2 + 3 * c2 ** 2 + 8 * c1 * c3 + 6 * c4) / 24

    p = (-1) ** L
    return int(round(0.5 * (_haar(lambda t: chiS(t, False) * _chi(L, t)) + p * _haar(lambda t: chiS(t, True) * _chi(L, t)))))


def _sym_rank(paths, L):
    rows = []
    for p in paths:
        T = path_tensor(p)
        acc = {}
        for idx in zip(*np.nonzero(np.abs(T) > 1e-13)):
            key = (idx[0] - L, tuple(sorted(lm_index(p.ls[j], idx[1 + j] - p.ls[j]) for j in range(p.nu))))
            acc[key] = acc.get(key, 0.0) + T[idx]
        rows.append(acc)
    keys = sorted(set(k for r in rows for k in r))
    return np.linalg.matrix_rank(np.array([[r.get(k, 0.0) for k in keys] for r in rows]), tol=1e-9)


@pytest.mark.parametrize("L,mult,n_paths", [(0, 23, 158), (1, 31, 284)])
def test_filtered_nu4_paths_are_complete(L, mult, n_paths):
    assert _sym4_multiplicity(L) == mult
    paths = enumerate_paths(3, 4, L)
    assert len(paths) == n_paths
    for p in paths:   # the filter: natural-parity intermediates
        s = p.ls[0]
        for j in range(1, 4):
            s += p.ls[j]
            assert (p.mids[j - 1] + s) % 2 == 0
    assert _sym_rank(paths, L) == mult


def test_nu4_tensor_equivariance():
    rng = np.random.default_rng(11)
    R = random_rotation(rng)
    D = {l: wigner_d_fit(l, R) for l in range(4)}
    for L in (0, 1):
        for p in enumerate_paths(3, 4, L)[::23]:
            T = path_tensor(p)
            lhs = np.einsum("Mabcd,ai,bj,ck,dl->Mijkl", T, D[p.ls[0]], D[p.ls[1]], D[p.ls[2]], D[p.ls[3]])
            rhs = np.einsum("MN,Nijkl->Mijkl", D[L], T)
            assert np.allclose(lhs, rhs, atol=1e-11)


def _inputs(prob, N=3, K=2, E=2, seed=0):
    rng = np.random.default_rng(seed)
    return rng.normal(size=(N, K, prob.n_lm)), rng.normal(size=(E, prob.n_paths, K)), rng.integers(0, E, N), rng


def test_corr4_bruteforce_rotation_inversion():
    prob = Problem(2, 4, [0, 1])          # lmax_in 2 keeps the 9^4 dense brute force small
    A, W, ne, rng = _inputs(prob, N=2, K=2)
    B = forward(prob, A, W, ne)
    assert np.abs(B - forward_bruteforce(prob, A, W, ne)).max() <= 1e-12 * np.abs(B).max()
    prob3 = Problem(3, 4, [0, 1])
    A, W, ne, rng = _inputs(prob3, N=2, K=2, seed=1)
    N, K = A.shape[:2]
    R = random_rotation(rng)
    B = forward(prob3, A, W, ne)
    Br = forward(prob3, np.einsum("ab,ikb->ika", block_diag_d(3, R), A), W, ne)
    D1 = wigner_d_fit(1, R)
    assert np.allclose(Br[:, :K], B[:, :K], atol=1e-10 * np.abs(B).max())                    # 0e invariant
    rot = np.einsum("MN,ikN->ikM", D1, B[:, K:].reshape(N, K, 3)).reshape(N, 3 * K)
    assert np.abs(Br[:, K:] - rot).max() <= 1e-10 * np.abs(B).max()                          # 1o rotates
    sgn = np.array([(-1) ** l for l in range(4) for _ in range(2 * l + 1)])
    Bi = forward(prob3, A * sgn, W, ne)
    assert np.allclose(Bi[:, :K], B[:, :K], atol=1e-12) and np.allclose(Bi[:, K:], -B[:, K:], atol=1e-12)


def test_corr4_homogeneity_isolates_nu4():
    prob = Problem(3, 4, [0])
    A, W, ne, _ = _inputs(prob, N=2, K=2, seed=2)
    W4 = W.copy()
    for p in prob.paths:
        if p.nu != 4:
            W4[:, p.col, :] = 0
    B4 = forward(prob, A, W4, ne)
    assert np.abs(B4).max() > 0
    assert np.allclose(forward(prob, 1.7 * A, W4, ne), 1.7 ** 4 * B4, rtol=1e-12, atol=1e-12)


def test_corr4_finite_differences_and_euler():
    prob = Problem(3, 4, [0, 1])
    A, W, ne, rng = _inputs(prob, N=2, K=2, seed=3)
    dB = rng.normal(size=(2, prob.out_dim(2)))
    dA, dW = backward(prob, A, W, ne, dB)
    h = 1e-6
    for _ in range(4):
        idx = tuple(rng.integers(0, s) for s in A.shape)
        Ap, Am = A.copy(), A.copy()
        Ap[idx] += h
        Am[idx] -= h
        fd = ((forward(prob, Ap, W, ne) - forward(prob, Am, W, ne)) * dB).sum() / (2 * h)
        assert fd == pytest.approx(dA[idx], rel=1e-6, abs=1e-7)
    B = forward(prob, A, W, ne)
    assert (W * dW).sum() == pytest.approx((dB * B).sum(), rel=1e-12)
    N, K = 2, 2
    lhs = (A * dA).sum(-1)
    rhs = np.zeros((N, K))
    for nu in (1, 2, 3, 4):
        Wn = W.copy()
        for p in prob.paths:
            if p.nu != nu:
                Wn[:, p.col, :] = 0
        Bn = forward(prob, A, Wn, ne)
        off = 0
        for L in prob.out_L:
            d = 2 * L + 1
            rhs += nu * (dB[:, off:off + K * d] * Bn[:, off:off + K * d]).reshape(N, K, d).sum(-1)
            off += K * d
    assert np.allclose(lhs, rhs, rtol=1e-10, atol=1e-10)


def test_corr4_c_evaluator_equals_python():
    from oracle.ceval import OracleC
    prob = Problem(3, 4, [0, 1])
    A, W, ne, rng = _inputs(prob, N=4, K=3, E=2, seed=4)
    A, W = A.astype(np.float32).astype(np.float64), W.astype(np.float32).astype(np.float64)
    dB = rng.normal(size=(4, prob.out_dim(3))).astype(np.float32).astype(np.float64)
    oc = OracleC(prob)
    assert np.allclose(oc.forward(A, W, ne), forward(prob, A, W, ne), rtol=1e-12, atol=1e-12)
    dA, dW = oc.backward(A, W, ne, dB)
    rA, rW = backward(prob, A, W, ne, dB)
    assert np.allclose(dA, rA, rtol=1e-11, atol=1e-11) and np.allclose(dW, rW, rtol=1e-11, atol=1e-11)

"""Pins for oracle/contraction.py (brute force, special cases, invariants, FD, identities)."""
import numpy as np
import pytest

from oracle.contraction import Problem, forward, backward, forward_bruteforce, path_features
from oracle.so3 import block_diag_d, random_rotation, wigner_d_fit, real_cg


def _inputs(prob, N=6, K=3, E=2, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(N, K, prob.n_lm))
    W = rng.normal(size=(E, prob.n_paths, K))
    ne = rng.integers(0, E, N)
    return A, W, ne, rng


def test_bruteforce_matches_sparse():
    prob = Problem(3, 3, [0, 1])
    A, W, ne, _ = _inputs(prob, N=3, K=2)
    B = forward(prob, A, W, ne)
    Bb = forward_bruteforce(prob, A, W, ne)
    assert np.abs(B - Bb).max() <= 1e-12 * np.abs(Bb).max()


def test_nu1_is_linear_map():
    prob = Problem(3, 1, [0, 1, 2, 3])
    A, W, ne, _ = _inputs(prob)
    B = forward(prob, A, W, ne)
    N, K = A.shape[:2]
    off = 0
    for c, L in enumerate(prob.out_L):
        blk = B[:, off:off + K * (2 * L + 1)].reshape(N, K, 2 * L + 1)
        expect = W[ne][:, c, :][:, :, None] * A[:, :, L * L:(L + 1) ** 2]
        assert np.allclose(blk, expect, atol=1e-14)
        off += K * (2 * L + 1)


@pytest.mark.parametrize("l", [1, 2, 3])
def test_corr2_scalar_closed_form(l):
    # only block l of A nonzero, out 0e, corr 2: B = W[(0,2,eta=l)] * sum_m A_lm^2 / sqrt(2l+1)
    prob = Problem(3, 2, [0])
    A, W, ne, _ = _inputs(prob)
    mask = np.zeros(16)
    mask[l * l:(l + 1) ** 2] = 1
    A = A * mask
    B = forward(prob, A, W, ne)
    col = 1 + l   # column 0 is (nu=1); nu=2 paths for L=0 are (0,0),(1,1),(2,2),(3,3)
    assert prob.paths[col].ls == (l, l)
    expect = W[ne][:, col, :] * (A ** 2).sum(-1) / np.sqrt(2 * l + 1)
    assert np.allclose(B, expect, atol=1e-13)


def test_homogeneity_isolates_orders():
    prob = Problem(3, 3, [0, 1])
    A, W, ne, _ = _inputs(prob)
    s = np.array([0.5, 1.0, 2.0])
    Bs = np.stack([forward(prob, si * A, W, ne) for si in s])
    V = np.stack([s ** nu for nu in (1, 2, 3)], 1)          # B(sA) = sum_nu s^nu B_nu
    Bnu = np.linalg.solve(V, Bs.reshape(3, -1)).reshape(Bs.shape)
    for nu in (1, 2, 3):
        Wn = W.copy()
        for p in prob.paths:
            if p.nu != nu:
                Wn[:, p.col, :] = 0
        assert np.allclose(Bnu[nu - 1], forward(prob, A, Wn, ne), atol=1e-10)


def _rotate_out(prob, B, N, K, D):
    out, off = [], 0
    for L in prob.out_L:
        blk = B[:, off:off + K * (2 * L + 1)].reshape(N, K, 2 * L + 1)
        out.append(np.einsum("MN,ikN->ikM", D[L], blk).reshape(N, -1))
        off += K * (2 * L + 1)
    return np.concatenate(out, 1)


def test_rotation_equivariance():
    prob = Problem(3, 3, [0, 1, 2])
    A, W, ne, rng = _inputs(prob, N=4, K=2)
    N, K = A.shape[:2]
    for _ in range(50):
        R = random_rotation(rng)
        Dfull = block_diag_d(3, R)
        D = {L: wigner_d_fit(L, R) for L in prob.out_L}
        B = forward(prob, A, W, ne)
        Br = forward(prob, np.einsum("ab,ikb->ika", Dfull, A), W, ne)
        rhs = _rotate_out(prob, B, N, K, D)
        assert np.abs(Br - rhs).max() <= 1e-10 * np.abs(B).max()
        assert np.allclose(Br[:, :K], B[:, :K], atol=1e-10 * np.abs(B).max())   # L=0 invariant


def test_inversion_parity():
    prob = Problem(3, 3, [0, 1, 2])
    A, W, ne, _ = _inputs(prob)
    N, K = A.shape[:2]
    sgn = np.array([(-1) ** l for l in range(4) for _ in range(2 * l + 1)])
    B = forward(prob, A, W, ne)
    Bi = forward(prob, A * sgn, W, ne)
    off = 0
    for L in prob.out_L:
        d = K * (2 * L + 1)
        assert np.allclose(Bi[:, off:off + d], (-1) ** L * B[:, off:off + d], atol=1e-12)
        off += d


def test_linearity_in_W_and_element_isolation():
    prob = Problem(3, 3, [0, 1])
    A, W, ne, rng = _inputs(prob, N=8, E=3)
    W2 = rng.normal(size=W.shape)
    assert np.allclose(forward(prob, A, 2 * W - W2, ne), 2 * forward(prob, A, W, ne) - forward(prob, A, W2, ne))
    Wc = W.copy()
    Wc[1] += 5.0
    B0, B1 = forward(prob, A, W, ne), forward(prob, A, Wc, ne)
    keep = ne != 1
    assert np.array_equal(B0[keep], B1[keep]) and not np.allclose(B0[~keep], B1[~keep])


def test_zero_in_zero_out_and_bad_element():
    prob = Problem(3, 3, [0])
    A, W, ne, _ = _inputs(prob)
    assert np.all(forward(prob, 0 * A, W, ne) == 0)
    ne2 = ne.copy()
    ne2[0] = W.shape[0]
    with pytest.raises(ValueError):
        forward(prob, A, W, ne2)


def test_finite_differences():
    prob = Problem(3, 3, [0, 1])
    for seed in range(20):
        A, W, ne, rng = _inputs(prob, N=2, K=2, seed=seed)
        dB = rng.normal(size=(2, prob.out_dim(2)))
        dA, dW = backward(prob, A, W, ne, dB)
        h = 1e-6
        for _ in range(3):
            idx = tuple(rng.integers(0, s) for s in A.shape)
            Ap, Am = A.copy(), A.copy()
            Ap[idx] += h
            Am[idx] -= h
            fd = ((forward(prob, Ap, W, ne) - forward(prob, Am, W, ne)) * dB).sum() / (2 * h)
            assert fd == pytest.approx(dA[idx], rel=1e-7, abs=1e-8)
            idx = tuple(rng.integers(0, s) for s in W.shape)
            Wp, Wm = W.copy(), W.copy()
            Wp[idx] += h
            Wm[idx] -= h
            fd = ((forward(prob, A, Wp, ne) - forward(prob, A, Wm, ne)) * dB).sum() / (2 * h)
            assert fd == pytest.approx(dW[idx], rel=1e-7, abs=1e-8)


def test_euler_and_weight_identities():
    prob = Problem(3, 3, [0, 1, 2])
    A, W, ne, rng = _inputs(prob, N=5, K=3)
    dB = rng.normal(size=(5, prob.out_dim(3)))
    dA, dW = backward(prob, A, W, ne, dB)
    B = forward(prob, A, W, ne)
    assert (W * dW).sum() == pytest.approx((dB * B).sum(), rel=1e-12)      # <W,dW> = <dB,B>
    # Euler: sum_a A_a dA_a = sum_nu nu <dB, B_nu>  per (node, channel)
    N, K = 5, 3
    lhs = (A * dA).sum(-1)
    rhs = np.zeros((N, K))
    for nu in (1, 2, 3):
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
    assert np.allclose(lhs, rhs, rtol=1e-11, atol=1e-11)


def test_onehot_dB_gives_path_features():
    prob = Problem(3, 3, [0, 1])
    A, W, ne, _ = _inputs(prob, N=3, K=2)
    P = path_features(prob, A)
    i, k, L, M = 1, 1, 1, -1
    dB = np.zeros((3, prob.out_dim(2)))
    dB[i, prob.out_off[L] * 2 + k * (2 * L + 1) + M + L] = 1.0
    _, dW = backward(prob, A, W, ne, dB)
    for p in prob.paths:
        expect = P[i, k, p.col, M + p.L] if p.L == L else 0.0
        assert dW[ne[i], p.col, k] == pytest.approx(expect, abs=1e-14)
    others = [z for z in range(W.shape[0]) if z != ne[i]]
    assert np.all(dW[others] == 0)


def test_backward2_against_finite_differences():
    """The double backward is the derivative of <uA, dA(A, W, dB)>: check it by central differences of
    the (already FD-pinned) backward; dB enters linearly, so its derivative is exact."""
    from oracle.contraction import backward2
    prob = Problem(3, 3, [0, 1])
    for seed in range(6):
        A, W, ne, rng = _inputs(prob, N=2, K=2, seed=seed)
        dB = rng.normal(size=(2, prob.out_dim(2)))
        uA = rng.normal(size=A.shape)
        dB_bar, A_bar, W_bar = backward2(prob, A, W, ne, dB, uA)
        f = lambda A_, W_, dB_: (uA * backward(prob, A_, W_, ne, dB_)[0]).sum()
        h = 1e-6
        for _ in range(3):
            idx = tuple(rng.integers(0, s) for s in A.shape)
            Ap, Am = A.copy(), A.copy()
            Ap[idx] += h
            Am[idx] -= h
            assert (f(Ap, W, dB) - f(Am, W, dB)) / (2 * h) == pytest.approx(A_bar[idx], rel=1e-7, abs=1e-8)
            idx = tuple(rng.integers(0, s) for s in W.shape)
            Wp, Wm = W.copy(), W.copy()
            Wp[idx] += h
            Wm[idx] -= h
            assert (f(A, Wp, dB) - f(A, Wm, dB)) / (2 * h) == pytest.approx(W_bar[idx], rel=1e-7, abs=1e-8)
            idx = tuple(rng.integers(0, s) for s in dB.shape)
            e = np.zeros_like(dB)
            e[idx] = 1.0
            assert f(A, W, e) == pytest.approx(dB_bar[idx], rel=1e-10, abs=1e-12)   # linear in dB


def test_backward2_jvp_and_symmetry():
    """dB_bar is the JVP of the forward in direction uA; <v, A_bar(uA)> = <uA, A_bar(v)> (the
    dB-weighted Hessian is symmetric)."""
    from oracle.contraction import backward2
    prob = Problem(3, 3, [0, 1, 2])
    A, W, ne, rng = _inputs(prob, N=3, K=2)
    dB = rng.normal(size=(3, prob.out_dim(2)))
    u, v = rng.normal(size=A.shape), rng.normal(size=A.shape)
    dB_bar, Au, _ = backward2(prob, A, W, ne, dB, u)
    _, Av, _ = backward2(prob, A, W, ne, dB, v)
    h = 1e-6
    jvp = (forward(prob, A + h * u, W, ne) - forward(prob, A - h * u, W, ne)) / (2 * h)
    assert np.allclose(jvp, dB_bar, rtol=1e-7, atol=1e-8)
    assert (v * Au).sum() == pytest.approx((u * Av).sum(), rel=1e-11)

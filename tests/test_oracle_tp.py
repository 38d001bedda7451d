"""Pins of the channelwise-TP oracle (oracle/tp.py; Alg. 2, Eq. (1) pooling)."""
import numpy as np
import pytest

from oracle.so3 import block_diag_d, random_rotation, real_sph_harm, wigner_d_fit
from oracle.tp import TPProblem, backward, forward, forward_bruteforce


def _graph(rng, N, E):
    sender = rng.integers(0, N, E)
    receiver = rng.integers(0, N, E)
    return sender, receiver


def _inputs(prob, N, E, K, seed=0, unit_y=True):
    rng = np.random.default_rng(seed)
    r = rng.normal(size=(E, 3))
    Y = real_sph_harm(prob.lmax_y, r / np.linalg.norm(r, axis=1, keepdims=True)) if unit_y else rng.normal(size=(E, prob.n_y))
    h = rng.normal(size=(N, prob.n_h, K))
    R = rng.normal(size=(E, prob.n_paths, K))
    s, t = _graph(rng, N, E)
    return Y, h, R, s, t, r, rng


def test_path_counts_and_parity():
    # MACE-MP layer-2 shape: Y up to l=3, hidden 0e+1o, A up to l=3 -> 4 + 6 paths
    prob = TPProblem(3, (0, 1), 3)
    assert prob.n_paths == 10
    assert all((l1 + l2 + l3) % 2 == 0 and abs(l1 - l2) <= l3 <= l1 + l2 for l1, l2, l3 in map(prob.path_l, range(10)))
    assert [prob.path_l(p) for p in range(4)] == [(0, 0, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0)]
    # scalar hidden features (layer 1): one path per Y order
    p0 = TPProblem(3, (0,), 3)
    assert [p0.path_l(p) for p in range(p0.n_paths)] == [(l, 0, l) for l in range(4)]


def test_bruteforce_loops_agree():
    prob = TPProblem(2, (0, 1, 2), 2)
    Y, h, R, s, t, _, _ = _inputs(prob, 5, 11, 3, unit_y=False)
    assert np.abs(forward(prob, Y, h, R, s, t, 5) - forward_bruteforce(prob, Y, h, R, s, t, 5)).max() < 1e-12


def test_scalar_paths_closed_forms():
    """(0, l, l): Y_00 R h_l (the coupling 0 x l -> l is the identity); (l, l, 0): R Y_l.h_l/sqrt(2l+1)."""
    rng = np.random.default_rng(1)
    N, E, K = 4, 9, 2
    prob = TPProblem(0, (2,), 2)          # single path (0, 2, 2)
    Y = rng.normal(size=(E, 1))
    h = rng.normal(size=(N, 5, K))
    R = rng.normal(size=(E, 1, K))
    s, t = _graph(rng, N, E)
    ref = np.zeros((N, K, 9))
    for e in range(E):
        ref[t[e], :, 4:9] += R[e, 0, :, None] * Y[e, 0] * h[s[e]].T
    assert np.abs(forward(prob, Y, h, R, s, t, N) - ref).max() < 1e-12
    prob = TPProblem(2, (2,), 0)          # single path (2, 2, 0)
    Y = rng.normal(size=(E, 9))
    ref = np.zeros((N, K, 1))
    for e in range(E):
        ref[t[e], :, 0] += R[e, 0, :] * (h[s[e]].T @ Y[e, 4:9]) / np.sqrt(5)
    assert np.abs(forward(prob, Y, h, R, s, t, N) - ref).max() < 1e-12


def test_vector_paths_closed_forms():
    """(1, 0, 1): R h_0 Y_1 (identity coupling); (1, 1, 2) applied to Y_1(u) x Y_1(u) is a fixed
    multiple of Y_2(u) (products of harmonics of one direction decompose into harmonics; scipy SH
    only); the axial (1, 1, 1) path is excluded by natural parity."""
    prob = TPProblem(1, (0, 1), 2)
    assert (1, 1, 1) not in [prob.path_l(p) for p in range(prob.n_paths)]
    rng = np.random.default_rng(2)
    u = rng.normal(size=(6, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    Y = real_sph_harm(1, u)                                 # [6][4]
    h = np.zeros((6, prob.n_h, 1))
    h[:, 0, 0] = rng.normal(size=6)                         # scalar block
    h[:, 1:4, 0] = Y[:, 1:4]                                # vector block = Y_1(u)
    paths = [prob.path_l(p) for p in range(prob.n_paths)]
    R = np.zeros((6, prob.n_paths, 1))
    R[:, paths.index((1, 0, 1)), 0] = 1.0
    A = forward(prob, Y, h, R, np.arange(6), np.arange(6), 6)
    assert np.abs(A[:, 0, 1:4] - h[:, 0, 0, None] * Y[:, 1:4]).max() < 1e-12
    R[:] = 0.0
    R[:, paths.index((1, 1, 2)), 0] = 1.0
    A2 = forward(prob, Y, h, R, np.arange(6), np.arange(6), 6)[:, 0, 4:9]
    Y2 = real_sph_harm(2, u)[:, 4:9]
    ratio = (A2 * Y2).sum(1) / (Y2 * Y2).sum(1)
    assert np.abs(A2 - ratio[:, None] * Y2).max() < 1e-12 and np.ptp(ratio) < 1e-12 and abs(ratio[0]) > 0.1


def test_rotation_equivariance():
    """Rotating the edge vectors and the hidden features rotates A (Wigner-D fitted from SH only)."""
    prob = TPProblem(3, (0, 1, 2), 3)
    N, E, K = 6, 20, 2
    Y, h, R, s, t, r, rng = _inputs(prob, N, E, K, seed=3)
    A = forward(prob, Y, h, R, s, t, N)
    for _ in range(3):
        Rot = random_rotation(rng)
        rr = r @ Rot.T
        Yr = real_sph_harm(3, rr / np.linalg.norm(rr, axis=1, keepdims=True))
        Dh = np.zeros((prob.n_h, prob.n_h))
        for b, l in enumerate(prob.hidden_l):
            o = prob.h_off[b]
            Dh[o:o + 2 * l + 1, o:o + 2 * l + 1] = wigner_d_fit(l, Rot)
        hr = np.einsum("ab,nbk->nak", Dh, h)
        Ar = forward(prob, Yr, hr, R, s, t, N)
        assert np.abs(Ar - np.einsum("ab,nkb->nka", block_diag_d(3, Rot), A)).max() < 1e-9 * np.abs(A).max()


def test_pooling_is_the_incidence_matrix_product_and_isolated_nodes():
    prob = TPProblem(2, (0, 1), 2)
    N, E, K = 7, 15, 3
    Y, h, R, s, t, _, _ = _inputs(prob, N, E, K, seed=4)
    t = np.where(t == 6, 0, t)            # node 6 receives nothing
    from oracle.tp import messages
    M = messages(prob, Y, h, R, s)
    inc = np.zeros((N, E))
    inc[t, np.arange(E)] = 1.0
    A = forward(prob, Y, h, R, s, t, N)
    assert np.abs(A - np.einsum("ne,ekc->nkc", inc, M)).max() < 1e-12
    assert not A[6].any()
    assert not forward(prob, Y[:0], h, R[:0], s[:0], t[:0], N).any()


def test_multilinearity():
    prob = TPProblem(2, (0, 1, 2), 2)
    N, E, K = 5, 12, 2
    Y, h, R, s, t, _, rng = _inputs(prob, N, E, K, seed=5, unit_y=False)
    f = lambda Y_, h_, R_: forward(prob, Y_, h_, R_, s, t, N)
    a, b = 0.7, -1.3
    for i, X in enumerate((Y, h, R)):
        X2 = rng.normal(size=X.shape)
        args1, args2, args3 = [Y, h, R], [Y, h, R], [Y, h, R]
        args1[i], args2[i], args3[i] = a * X + b * X2, X, X2
        assert np.abs(f(*args1) - a * f(*args2) - b * f(*args3)).max() < 1e-11


def test_backward_finite_differences_and_euler_identities():
    prob = TPProblem(2, (0, 1), 2)
    N, E, K = 5, 13, 2
    Y, h, R, s, t, _, rng = _inputs(prob, N, E, K, seed=6, unit_y=False)
    dA = rng.normal(size=(N, K, prob.n_out))
    dY, dh, dR = backward(prob, Y, h, R, s, t, N, dA)
    A = forward(prob, Y, h, R, s, t, N)
    # A is linear in each of Y, h, R separately: <dA, A> = <dY, Y> = <dh, h> = <dR, R>
    v = (dA * A).sum()
    for g, x in ((dY, Y), (dh, h), (dR, R)):
        assert (g * x).sum() == pytest.approx(v, rel=1e-11)
    f = lambda Y_, h_, R_: (dA * forward(prob, Y_, h_, R_, s, t, N)).sum()
    eps = 1e-6
    for i, (X, G) in enumerate(((Y, dY), (h, dh), (R, dR))):
        for _ in range(4):
            idx = tuple(rng.integers(0, n) for n in X.shape)
            Xp, Xm = X.copy(), X.copy()
            Xp[idx] += eps
            Xm[idx] -= eps
            ap, am = [Y, h, R], [Y, h, R]
            ap[i], am[i] = Xp, Xm
            assert (f(*ap) - f(*am)) / (2 * eps) == pytest.approx(G[idx], rel=1e-7, abs=1e-7)


def test_double_backward_composition_by_finite_differences():
    """The TP is linear in each of Y, h, R, so the derivatives of <(uY, uh, uR), backward(Y, h, R, dA)>
    are TP passes with one input replaced by its cotangent (ops._TPBwdFn): pinned here against
    central differences of the oracle backward."""
    prob = TPProblem(2, (0, 1), 2)
    N, E, K = 5, 12, 2
    Y, h, R, s, t, _, rng = _inputs(prob, N, E, K, seed=8, unit_y=False)
    dA = rng.normal(size=(N, K, prob.n_out))
    uY, uh, uR = rng.normal(size=Y.shape), rng.normal(size=h.shape), rng.normal(size=R.shape)

    def L(Y_, h_, R_, dA_):
        gY, gh, gR = backward(prob, Y_, h_, R_, s, t, N, dA_)
        return (uY * gY).sum() + (uh * gh).sum() + (uR * gR).sum()

    dA_bar = forward(prob, uY, h, R, s, t, N) + forward(prob, Y, uh, R, s, t, N) + forward(prob, Y, h, uR, s, t, N)
    aY, _, aR = backward(prob, Y, uh, R, s, t, N, dA)
    bY, bh, _ = backward(prob, Y, h, uR, s, t, N, dA)
    _, ch, cR = backward(prob, uY, h, R, s, t, N, dA)
    comp = {0: aY + bY, 1: bh + ch, 2: aR + cR, 3: dA_bar}
    eps = 1e-6
    args = [Y, h, R, dA]
    for i in range(4):
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in args[i].shape)
            ap, am = [a.copy() for a in args], [a.copy() for a in args]
            ap[i][idx] += eps
            am[i][idx] -= eps
            assert (L(*ap) - L(*am)) / (2 * eps) == pytest.approx(comp[i][idx], rel=1e-6, abs=1e-6)

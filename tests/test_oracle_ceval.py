"""The C fp64 evaluator (timing / full-size oracle) against the Python oracle."""
import numpy as np

from oracle.contraction import Problem, forward, backward
from oracle.ceval import OracleC


def test_ceval_matches_python():
    for out_L, corr in (((0,), 3), ((0, 1), 3), ((0, 1, 2), 3), ((1,), 2)):
        prob = Problem(3, corr, out_L)
        oc = OracleC(prob)
        rng = np.random.default_rng(7)
        N, K, E = 20, 4, 3
        A = rng.normal(size=(N, K, 16)).astype(np.float32)
        W = rng.normal(size=(E, prob.n_paths, K)).astype(np.float32)
        ne = rng.integers(0, E, N).astype(np.int32)
        B = forward(prob, A, W, ne)
        assert np.abs(oc.forward(A, W, ne) - B).max() <= 1e-13 * np.abs(B).max()
        dB = rng.normal(size=B.shape).astype(np.float32)
        dA, dW = backward(prob, A, W, ne, dB)
        dAc, dWc = oc.backward(A, W, ne, dB)
        assert np.abs(dAc - dA).max() <= 1e-13 * np.abs(dA).max()
        assert np.abs(dWc - dW).max() <= 1e-13 * np.abs(dW).max()


def test_ceval_backward2_matches_python():
    from oracle.contraction import backward2
    for out_L, corr in (((0, 1), 3), ((0, 1, 2), 3), ((1,), 2)):
        prob = Problem(3, corr, out_L)
        oc = OracleC(prob)
        rng = np.random.default_rng(11)
        N, K, E = 12, 3, 3
        A = rng.normal(size=(N, K, 16)).astype(np.float32)
        W = rng.normal(size=(E, prob.n_paths, K)).astype(np.float32)
        ne = rng.integers(0, E, N).astype(np.int32)
        dB = rng.normal(size=(N, prob.out_dim(K))).astype(np.float32)
        uA = rng.normal(size=A.shape).astype(np.float32)
        ref = backward2(prob, A, W, ne, dB, uA)
        got = oc.backward2(A, W, ne, dB, uA)
        for r, g in zip(ref, got):
            assert np.abs(g - r).max() <= 1e-13 * np.abs(r).max()

"""Alg. 3 forward and backward, fp64 (oracle; test infrastructure only).

Forward (Eq. (2); API name "B" = the
paper's m, reading s1):

    B[i, k, (L, M)] = sum_nu sum_eta W[z_i, (L,nu,eta), k]
                      * sum_{(M, t) in nnz U_{nu,L,eta}} U[M, t] * prod_j A[i, k, t_j]

Backward (forces are "derivatives of the total energy"):

    dA[i,k,a]  = sum_{L,M} dB[i,k,(L,M)] sum_{paths} W[z_i,p,k] sum_{nnz} U
                 * sum_{j: t_j = a} prod_{j' != j} A[i,k,t_j']
    dW[z,p,k]  = sum_{i: z_i = z} sum_M dB[i,k,(L,M)] sum_{nnz} U prod_j A[i,k,t_j]

Layouts: A, dA [N][K][(lmax+1)^2] (lm fastest); W, dW
[E][P][K] with P = number of paths; B, dB [N][sum_L K(2L+1)], per-L block
[K][2L+1] (m fastest), blocks in out_L order. node_elem int [N] in [0, E).

Everything loops over the raw ordered tuples (no symmetrization, no folding),
vectorized over (node, channel) with numpy.
"""
import numpy as np

from .paths import build_paths, dense_U


class Problem:
    """Tables for one (lmax_in, correlation, out_L)."""

    def __init__(self, lmax_in, correlation, out_L):
        self.lmax_in, self.correlation, self.out_L = lmax_in, correlation, tuple(out_L)
        self.paths = build_paths(lmax_in, correlation, out_L)
        self.n_paths = len(self.paths)
        self.n_lm = (lmax_in + 1) ** 2
        self.out_off = {}
        off = 0
        for L in self.out_L:
            self.out_off[L] = off
            off += 2 * L + 1
        self.out_per_channel = off

    def out_dim(self, K):
        return K * self.out_per_channel

    def block_sizes(self):
        """[(L, nu, n_eta)] in W column order (for W initialization)."""
        out = []
        for p in self.paths:
            if out and out[-1][0] == p.L and out[-1][1] == p.nu:
                out[-1] = (p.L, p.nu, out[-1][2] + 1)
            else:
                out.append((p.L, p.nu, 1))
        return out


def _check(prob, A, W, node_elem):
    N, K, n = A.shape
    assert n == prob.n_lm
    E, P, K2 = W.shape
    assert P == prob.n_paths and K2 == K
    node_elem = np.asarray(node_elem)
    if N and (node_elem.min() < 0 or node_elem.max() >= E):
        raise ValueError("species index without weights")  # SPEC.md:363 / DESIGN.md §4
    return N, K, E


def _prod(A, ts, skip=-1):
    out = np.ones(A.shape[:2])
    for j, t in enumerate(ts):
        if j != skip:
            out = out * A[:, :, t]
    return out


def forward(prob, A, W, node_elem):
    A = np.asarray(A, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    N, K, E = _check(prob, A, W, node_elem)
    Wn = W[np.asarray(node_elem)]                     # [N][P][K] per-node weights
    out = {L: np.zeros((N, K, 2 * L + 1)) for L in prob.out_L}
    for p in prob.paths:
        w = Wn[:, p.col, :]
        for M, ts, u in p.terms:
            out[p.L][:, :, M + p.L] += w * u * _prod(A, ts)
    return np.concatenate([out[L].reshape(N, -1) for L in prob.out_L], axis=1)


def _split_out(prob, X, N, K):
    res, off = {}, 0
    for L in prob.out_L:
        d = K * (2 * L + 1)
        res[L] = np.asarray(X[:, off:off + d], dtype=np.float64).reshape(N, K, 2 * L + 1)
        off += d
    return res


def backward(prob, A, W, node_elem, dB):
    A = np.asarray(A, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    N, K, E = _check(prob, A, W, node_elem)
    node_elem = np.asarray(node_elem)
    Wn = W[node_elem]
    g = _split_out(prob, dB, N, K)
    dA = np.zeros_like(A)
    dW = np.zeros_like(W)
    for p in prob.paths:
        w = Wn[:, p.col, :]
        P = np.zeros((N, K))                           # sum_M dB * (path feature)
        for M, ts, u in p.terms:
            gM = g[p.L][:, :, M + p.L]
            P += gM * u * _prod(A, ts)
            for j, t in enumerate(ts):
                dA[:, :, t] += gM * w * u * _prod(A, ts, skip=j)
        for z in range(E):
            sel = node_elem == z
            if sel.any():
                dW[z, p.col, :] = P[sel].sum(axis=0)
    return dA, dW


def path_features(prob, A):
    """P[i, k, path, M] = sum_{nnz} U prod A  (the paper's B_{eta,kLM}, reading s1)."""
    A = np.asarray(A, dtype=np.float64)
    N, K, _ = A.shape
    Lmax = max(prob.out_L)
    P = np.zeros((N, K, prob.n_paths, 2 * Lmax + 1))
    for p in prob.paths:
        for M, ts, u in p.terms:
            P[:, :, p.col, M + p.L] += u * _prod(A, ts)
    return P


def forward_bruteforce(prob, A, W, node_elem):
    """Dense U over all (lmax+1)^(2 nu) tuples, one node/channel at a time (tiny only)."""
    A = np.asarray(A, dtype=np.float64)
    N, K, _ = A.shape
    dense = [(p, dense_U(p, prob.lmax_in)) for p in prob.paths]
    out = {L: np.zeros((N, K, 2 * L + 1)) for L in prob.out_L}
    letters = "abcd"
    for i in range(N):
        z = node_elem[i]
        for k in range(K):
            a = A[i, k]
            for p, U in dense:
                spec = "M" + letters[:p.nu] + "," + ",".join(letters[:p.nu]) + "->M"
                out[p.L][i, k] += W[z, p.col, k] * np.einsum(spec, U, *([a] * p.nu))
    return np.concatenate([out[L].reshape(N, -1) for L in prob.out_L], axis=1)


def backward2(prob, A, W, node_elem, dB, uA):
    """Double backward: derivatives of <uA, dA(A, W, dB)> w.r.t. A, W and dB (forces in the loss,
    PAPER.md:331, 967, 1549), from the raw ordered tuples:

        dB_bar[i,k,(L,M)] = sum_{paths} W sum_{nnz} U sum_j uA[t_j] prod_{j' != j} A[t_j']
        W_bar[z,p,k]      = sum_{i: z_i = z} sum_M dB_M sum_{nnz} U sum_j uA[t_j] prod_{j' != j} A[t_j']
        A_bar[i,k,b]      = sum_M dB_M sum_{paths} W sum_{nnz} U sum_{j} uA[t_j]
                            sum_{j'' != j, t_j'' = b} prod_{j' not in {j, j''}} A[t_j']
    """
    A = np.asarray(A, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    uA = np.asarray(uA, dtype=np.float64)
    N, K, E = _check(prob, A, W, node_elem)
    node_elem = np.asarray(node_elem)
    Wn = W[node_elem]
    g = _split_out(prob, dB, N, K)
    dB_bar = {L: np.zeros((N, K, 2 * L + 1)) for L in prob.out_L}
    A_bar = np.zeros_like(A)
    W_bar = np.zeros_like(W)

    def prod_except(ts, skip):
        out = np.ones(A.shape[:2])
        for jj, t in enumerate(ts):
            if jj not in skip:
                out = out * A[:, :, t]
        return out

    for p in prob.paths:
        w = Wn[:, p.col, :]
        Pp = np.zeros((N, K))
        for M, ts, u in p.terms:
            gM = g[p.L][:, :, M + p.L]
            jvp = np.zeros((N, K))                       # sum_j uA[t_j] prod_{j' != j} A
            for j, t in enumerate(ts):
                jvp += uA[:, :, t] * prod_except(ts, {j})
            dB_bar[p.L][:, :, M + p.L] += w * u * jvp
            Pp += gM * u * jvp
            for j, t in enumerate(ts):
                for j2, b in enumerate(ts):
                    if j2 != j:
                        A_bar[:, :, b] += gM * w * u * uA[:, :, t] * prod_except(ts, {j, j2})
        for z in range(E):
            sel = node_elem == z
            if sel.any():
                W_bar[z, p.col, :] = Pp[sel].sum(axis=0)
    dB_bar = np.concatenate([dB_bar[L].reshape(N, -1) for L in prob.out_L], axis=1)
    return dB_bar, A_bar, W_bar

"""Channelwise tensor product + edge->node sum (Alg. 2, pooling PAPER.md:321-324
Eq. (1) and PAPER.md:592) -- ORACLE, test infrastructure only (see oracle/__init__.py).

Alg. 2, line 6, per edge ji (sender j, receiver i) and channel k:

    A_{ji,k,l3 m3} += C^{l3 m3}_{l1 m1, l2 m2} R_{ji,k,l1 l2 l3} Y^{m1}_{ji,l1} h_{j,k,l2 m2}

summed over all (l1 m1, l2 m2) (line 5), and the messages are pooled onto the receiver with a
sum over its neighbours (Eq. (1) with the sum as the permutation-invariant pooling):

    A_{i,k,l3 m3} = sum_{j in N(i)} A_{ji,k,l3 m3}.

Readings (t1-t6):
  t1  C = the real coupling of oracle.so3.real_cg (the same normalization and sign rule as the
      contraction, readings s7/s8); a path is one (l1, l2, l3) with the triangle rule and
      natural parity (l1 + l2 + l3 even: Y_l1 has parity (-1)^l1, h_l2 (-1)^l2, and the output
      irrep l3 of the A feature row has natural parity, like the contraction's input).
  t2  paths ordered lexicographically by (l1, l2, l3); R has one weight per (edge, path,
      channel), channel fastest: R[E][P][K] (e3nn's per-instruction weight blocks).
  t3  h holds the hidden irreps `hidden_l` (strictly increasing l, one block of 2l+1
      components each), component-major with the channel fastest: h[N][n_h][K] (like R);
      Y[E][(lmax_y+1)^2] with lm = l^2 + l + m.
  t4  output A[N][K][(lmax_out+1)^2] (the contraction's input layout); nodes without incoming
      edges get A = 0; the linear mixing and 1/avg-neighbour scaling that MACE applies after the
      sum are outside the kernel ("after a further linear combination").
  t5  edges are (sender[e], receiver[e]) pairs; any order here (the product requires receiver-
      sorted edges and reports EINVAL otherwise).
  t6  the backward gives dY, dh, dR of <dA, A> (forces flow through Y).
"""
import numpy as np

from .so3 import real_cg


class TPProblem:
    def __init__(self, lmax_y, hidden_l, lmax_out):
        self.lmax_y, self.hidden_l, self.lmax_out = int(lmax_y), tuple(int(l) for l in hidden_l), int(lmax_out)
        assert all(a < b for a, b in zip(self.hidden_l, self.hidden_l[1:])), "hidden_l strictly increasing"
        self.n_y = (self.lmax_y + 1) ** 2
        self.n_out = (self.lmax_out + 1) ** 2
        self.h_off = []
        off = 0
        for l in self.hidden_l:
            self.h_off.append(off)
            off += 2 * l + 1
        self.n_h = off
        self.paths = []     # (l1, hidden block index, l3)
        for l1 in range(self.lmax_y + 1):
            for b, l2 in enumerate(self.hidden_l):
                for l3 in range(self.lmax_out + 1):
                    if abs(l1 - l2) <= l3 <= l1 + l2 and (l1 + l2 + l3) % 2 == 0:
                        self.paths.append((l1, b, l3))
        self.n_paths = len(self.paths)

    def path_l(self, p):
        l1, b, l3 = self.paths[p]
        return l1, self.hidden_l[b], l3

    def blocks(self, p):
        """(Y slice, h slice, A slice, C[m3, m1, m2]) of path p."""
        l1, b, l3 = self.paths[p]
        l2 = self.hidden_l[b]
        ys = slice(l1 * l1, (l1 + 1) ** 2)
        hs = slice(self.h_off[b], self.h_off[b] + 2 * l2 + 1)
        As = slice(l3 * l3, (l3 + 1) ** 2)
        return ys, hs, As, real_cg(l1, l2, l3)


def _check(prob, Y, h, R, sender, receiver, N):
    E = len(sender)
    K = h.shape[2]
    assert Y.shape == (E, prob.n_y) and h.shape == (N, prob.n_h, K) and R.shape == (E, prob.n_paths, K)
    assert len(receiver) == E
    return E, K


def messages(prob, Y, h, R, sender):
    """Per-edge messages A_{ji,k,l3m3} of Alg. 2, [E][K][n_out]."""
    Y, h, R = (np.asarray(x, dtype=np.float64) for x in (Y, h, R))
    sender = np.asarray(sender, dtype=np.int64)
    hs_all = h.transpose(0, 2, 1)[sender]                 # h_{j,k,.} of each edge's sender, [E][K][n_h]
    E, K = R.shape[0], R.shape[2]
    M = np.zeros((E, K, prob.n_out))
    for p in range(prob.n_paths):
        ys, hs, As, C = prob.blocks(p)
        # sum_{m1,m2} C[m3,m1,m2] Y[e,m1] h[e,k,m2], weighted by R[e,p,k]
        M[:, :, As] += R[:, p, :, None] * np.einsum("cab,ea,ekb->ekc", C, Y[:, ys], hs_all[:, :, hs])
    return M


def forward(prob, Y, h, R, sender, receiver, N):
    """A[N][K][n_out] = sum over edges into each node of the Alg. 2 messages (Eq. (1))."""
    E, K = _check(prob, np.asarray(Y), np.asarray(h), np.asarray(R), sender, receiver, N)
    A = np.zeros((N, K, prob.n_out))
    np.add.at(A, np.asarray(receiver, dtype=np.int64), messages(prob, Y, h, R, sender))
    return A


def backward(prob, Y, h, R, sender, receiver, N, dA):
    """(dY [E][n_y], dh [N][n_h][K], dR [E][P][K]) of <dA, forward(...)>."""
    Y, h, R, dA = (np.asarray(x, dtype=np.float64) for x in (Y, h, R, dA))
    E, K = _check(prob, Y, h, R, sender, receiver, N)
    sender = np.asarray(sender, dtype=np.int64)
    receiver = np.asarray(receiver, dtype=np.int64)
    g = dA[receiver]                                      # dA_{i,k,.} of each edge's receiver
    hs_all = h.transpose(0, 2, 1)[sender]
    dY = np.zeros_like(Y)
    dR = np.zeros_like(R)
    dhe = np.zeros((E, K, prob.n_h))                      # per-edge contribution to dh_{sender}
    for p in range(prob.n_paths):
        ys, hs, As, C = prob.blocks(p)
        v = np.einsum("cab,ea,ekb->ekc", C, Y[:, ys], hs_all[:, :, hs])
        dR[:, p, :] = np.einsum("ekc,ekc->ek", g[:, :, As], v)
        w = R[:, p, :, None] * g[:, :, As]                # R_p dA_{l3 m3}
        dY[:, ys] += np.einsum("cab,ekc,ekb->ea", C, w, hs_all[:, :, hs])
        dhe[:, :, hs] += np.einsum("cab,ekc,ea->ekb", C, w, Y[:, ys])
    dh = np.zeros((N, K, prob.n_h))
    np.add.at(dh, sender, dhe)
    return dY, dh.transpose(0, 2, 1).copy(), dR


def forward_bruteforce(prob, Y, h, R, sender, receiver, N):
    """Alg. 2 line by line in plain Python loops (tiny inputs only)."""
    E = len(sender)
    K = h.shape[2]
    A = np.zeros((N, K, prob.n_out))
    for e in range(E):
        j, i = int(sender[e]), int(receiver[e])
        for k in range(K):
            for p in range(prob.n_paths):
                l1, l2, l3 = prob.path_l(p)
                ys, hs, As, C = prob.blocks(p)
                for m3 in range(2 * l3 + 1):
                    for m1 in range(2 * l1 + 1):
                        for m2 in range(2 * l2 + 1):
                            A[i, k, As.start + m3] += (C[m3, m1, m2] * R[e, p, k] * Y[e, ys.start + m1]
                                                       * h[j, hs.start + m2, k])
    return A

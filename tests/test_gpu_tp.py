"""GPU parity of the channelwise tensor product (symcon_tp_*) against the
fp64 oracle (oracle/tp.py), element by element; tolerance as for the contraction: max|err| <=
1e-4 * max|ref| (north_star), gated at 1e-5 here."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _rel(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    s = np.abs(ref).max()
    return np.abs(x - ref).max() / (s if s > 0 else 1.0)


def _setup(lmax_y, hidden, lmax_out, K, sizes, deg=30, seed=0):
    from paper_2504_10700_b200.ops import ChannelwiseTP
    from synth.inputs import gen_tp_graph, gen_tp_inputs
    tp = ChannelwiseTP(lmax_y, hidden, lmax_out, K, device=0)
    s, r = gen_tp_graph(sizes, deg, seed)
    N, E = int(np.sum(sizes)), len(s)
    Y, h, R = gen_tp_inputs(N, E, K, tp.n_y, tp.n_h, tp.n_paths, "cuda", seed)
    return tp, Y, h, R, torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda(), N


def _host(*ts):
    return [t.detach().cpu().numpy() for t in ts]


@pytest.mark.parametrize("name,lmax_y,hidden,lmax_out,K,sizes", [
    ("mp_layer2", 3, (0, 1), 3, 128, [40, 25, 60, 31]),
    ("layer1_scalar", 3, (0,), 3, 64, [30, 12, 50]),
    ("hidden_012", 3, (0, 1, 2), 3, 32, [20, 33]),
    ("ragged_K13", 2, (0, 1), 2, 13, [17, 9, 30]),
    ("lmax_y1_out1", 1, (1,), 1, 40, [8, 8, 8]),
    ("hidden_0123", 3, (0, 1, 2, 3), 3, 33, [12, 20]),
    ("even_K6", 3, (0, 1), 3, 6, [9, 14]),            # channel pairs with 8-byte async chunks
    ("K96_ragged_pairs", 2, (0, 1), 2, 96, [20, 25]),  # last 64-channel group half full
    ("K1_scalar", 2, (0,), 2, 1, [5, 6]),
    ("Y_l0_only", 0, (0, 1, 2), 2, 16, [7, 9]),
])
def test_tp_against_oracle(name, lmax_y, hidden, lmax_out, K, sizes):
    from oracle.tp import TPProblem, forward, backward
    tp, Y, h, R, s, r, N = _setup(lmax_y, hidden, lmax_out, K, sizes)
    prob = TPProblem(lmax_y, hidden, lmax_out)
    assert tp.n_paths == prob.n_paths
    assert [tuple(int(x) for x in __import__("paper_2504_10700_b200")._lib.symcon_tp_path(tp.plan, p))
            for p in range(tp.n_paths)] == [prob.path_l(p) for p in range(prob.n_paths)]
    A = tp.forward_raw(Y, h, R, s, r)
    dA = torch.randn(A.shape, generator=torch.Generator("cuda").manual_seed(1), device="cuda")
    dY, dh, dR = tp.backward_raw(Y, h, R, s, r, dA)
    torch.cuda.synchronize()
    assert tp.check_device_error()[0] == 0
    hY, hh, hR, hs, hr, hdA = _host(Y, h, R, s, r, dA)
    assert _rel(A.cpu(), forward(prob, hY, hh, hR, hs, hr, N)) < TOL, name
    rY, rh, rR = backward(prob, hY, hh, hR, hs, hr, N, hdA)
    assert _rel(dY.cpu(), rY) < TOL, name
    assert _rel(dh.cpu(), rh) < TOL, name
    assert _rel(dR.cpu(), rR) < TOL, name


def test_tp_mid_size_mp_shape():
    """MP layer-2 shape on 2,000 nodes (~55k edges, degree 30 within 10-100-atom molecules)."""
    from oracle.tp import TPProblem, forward, backward
    from synth.inputs import molecule_sizes
    sizes = molecule_sizes(2000, seed=3)
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 128, sizes, seed=3)
    A = tp.forward_raw(Y, h, R, s, r)
    dA = torch.randn(A.shape, generator=torch.Generator("cuda").manual_seed(2), device="cuda")
    dY, dh, dR = tp.backward_raw(Y, h, R, s, r, dA)
    torch.cuda.synchronize()
    prob = TPProblem(3, (0, 1), 3)
    hY, hh, hR, hs, hr, hdA = _host(Y, h, R, s, r, dA)
    assert _rel(A.cpu(), forward(prob, hY, hh, hR, hs, hr, N)) < TOL
    rY, rh, rR = backward(prob, hY, hh, hR, hs, hr, N, hdA)
    for got, ref in ((dY, rY), (dh, rh), (dR, rR)):
        assert _rel(got.cpu(), ref) < TOL


def test_tp_edge_cases_and_errors():
    from paper_2504_10700_b200 import _lib
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 32, [10, 10])
    # isolated node: drop the edges into node 3 -> A[3] = 0, its dh still gets its out-edges
    keep = (r != 3)
    Yk, Rk, sk, rk = Y[keep].contiguous(), R[keep].contiguous(), s[keep].contiguous(), r[keep].contiguous()
    A = tp.forward_raw(Yk, h, Rk, sk, rk)
    torch.cuda.synchronize()
    assert torch.count_nonzero(A[3]) == 0 and torch.count_nonzero(A[4]) > 0
    # no edges at all: A = 0, dh = 0
    e0 = lambda *sh: torch.zeros(sh, device="cuda")
    i0 = torch.zeros(0, dtype=torch.int32, device="cuda")
    A0 = tp.forward_raw(e0(0, tp.n_y), h, e0(0, tp.n_paths, 32), i0, i0)
    dY0, dh0, dR0 = tp.backward_raw(e0(0, tp.n_y), h, e0(0, tp.n_paths, 32), i0, i0, torch.ones_like(A0))
    torch.cuda.synchronize()
    assert torch.count_nonzero(A0) == 0 and torch.count_nonzero(dh0) == 0 and dY0.numel() == 0
    # unsorted receivers -> EINVAL at the first offending edge; outputs unspecified but no fault
    r2 = r.clone()
    r2[5], r2[6] = r[6] + 1, r[5]
    tp.forward_raw(Y, h, R, s, r2)
    st, bad = tp.check_device_error()
    assert st == _lib.SYMCON_EINVAL and bad == 6
    # out-of-range sender -> EINVAL
    s2 = s.clone()
    s2[7] = N + 5
    tp.forward_raw(Y, h, R, s2, r)
    tp.backward_raw(Y, h, R, s2, r, torch.ones((N, 32, tp.n_out), device="cuda"))
    st, bad = tp.check_device_error()
    assert st == _lib.SYMCON_EINVAL and bad == 7
    # valid again afterwards
    tp.forward_raw(Y, h, R, s, r)
    assert tp.check_device_error()[0] == 0


def test_tp_deterministic_and_subsets():
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 64, [50, 40, 70])
    dA = torch.randn((N, 64, 16), generator=torch.Generator("cuda").manual_seed(3), device="cuda")
    a1 = tp.forward_raw(Y, h, R, s, r)
    g1 = tp.backward_raw(Y, h, R, s, r, dA)
    a2 = tp.forward_raw(Y, h, R, s, r)
    g2 = tp.backward_raw(Y, h, R, s, r, dA)
    assert torch.equal(a1, a2) and all(torch.equal(x, y) for x, y in zip(g1, g2))
    for mask in ((True, False, False), (False, True, False), (False, False, True)):
        part = tp.backward_raw(Y, h, R, s, r, dA, *mask)
        for m, full, x in zip(mask, g1, part):
            assert (x is None) != m and (x is None or torch.equal(x, full))


def test_tp_autograd_and_euler_identities():
    """Through autograd; A is linear in each of Y, h, R: <dA, A> = <dY, Y> = <dh, h> = <dR, R>."""
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 64, [30, 45])
    Yg, hg, Rg = (x.clone().requires_grad_(True) for x in (Y, h, R))
    A = tp(Yg, hg, Rg, s, r)
    dA = torch.randn(A.shape, generator=torch.Generator("cuda").manual_seed(4), device="cuda")
    (A * dA).sum().backward()
    v = (A.double() * dA.double()).sum().item()
    for g, x in ((Yg.grad, Y), (hg.grad, h), (Rg.grad, R)):
        assert abs((g.double() * x.double()).sum().item() - v) <= 1e-5 * (A.double().abs() * dA.double().abs()).sum().item()


def test_tp_full_size_sampled():
    """MP layer-2 shape at the bench size (50k nodes, ~1.46M edges): sampled receivers (A, and
    dY / dR of their incoming edges) and sampled senders (dh) against the oracle."""
    from oracle.tp import TPProblem, forward, backward
    from synth.inputs import molecule_sizes
    sizes = molecule_sizes(50_000, seed=0)
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 128, sizes, seed=0)
    A = tp.forward_raw(Y, h, R, s, r)
    dA = torch.randn(A.shape, generator=torch.Generator("cuda").manual_seed(5), device="cuda")
    dY, dh, dR = tp.backward_raw(Y, h, R, s, r, dA)
    torch.cuda.synchronize()
    assert tp.check_device_error()[0] == 0
    prob = TPProblem(3, (0, 1), 3)
    rng = np.random.default_rng(0)
    nodes = np.sort(rng.choice(N, 16, replace=False))
    hs, hr = _host(s, r)
    # receivers: their incoming edges only
    eidx = np.nonzero(np.isin(hr, nodes))[0]
    te = torch.from_numpy(eidx).cuda()
    hY, hh, hR, hdA = _host(Y[te], h, R[te], dA)
    Aref = forward(prob, hY, hh, hR, hs[eidx], hr[eidx], N)[nodes]
    assert _rel(A[torch.from_numpy(nodes).cuda()].cpu(), Aref) < TOL
    rY, _, rR = backward(prob, hY, hh, hR, hs[eidx], hr[eidx], N, hdA)
    assert _rel(dY[te].cpu(), rY) < TOL and _rel(dR[te].cpu(), rR) < TOL
    # senders: all their outgoing edges
    eidx = np.nonzero(np.isin(hs, nodes))[0]
    te = torch.from_numpy(eidx).cuda()
    hY, hR = _host(Y[te], R[te])
    _, rh, _ = backward(prob, hY, hh, hR, hs[eidx], hr[eidx], N, hdA)
    assert _rel(dh[torch.from_numpy(nodes).cuda()].cpu(), rh[nodes]) < TOL


def test_tp_double_backward_force_style_loss():
    """create_graph=True through the TP (forces flow through Y and R): loss = <dY, V1> + <dh, V2> +
    <dR, V3> of the gradients of <A, Rb>; its gradients against the oracle composition (pinned by
    finite differences in tests/test_oracle_tp.py)."""
    from oracle.tp import TPProblem, forward, backward
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 64, [20, 31], seed=4)
    g = torch.Generator("cuda").manual_seed(6)
    Rb = torch.randn((N, 64, tp.n_out), generator=g, device="cuda")
    V1, V2, V3 = (torch.randn(x.shape, generator=g, device="cuda") for x in (Y, h, R))
    Yg, hg, Rg, Rbg = (x.clone().requires_grad_(True) for x in (Y, h, R, Rb))
    A = tp(Yg, hg, Rg, s, r)
    gY, gh, gR = torch.autograd.grad((A * Rbg).sum(), (Yg, hg, Rg), create_graph=True)
    ((gY * V1).sum() + (gh * V2).sum() + (gR * V3).sum()).backward()
    torch.cuda.synchronize()
    prob = TPProblem(3, (0, 1), 3)
    hY, hh, hR, hs, hr, hRb, u1, u2, u3 = _host(Y, h, R, s, r, Rb, V1, V2, V3)
    dA_bar = forward(prob, u1, hh, hR, hs, hr, N) + forward(prob, hY, u2, hR, hs, hr, N) + forward(prob, hY, hh, u3, hs, hr, N)
    aY, _, aR = backward(prob, hY, u2, hR, hs, hr, N, hRb)
    bY, bh, _ = backward(prob, hY, hh, u3, hs, hr, N, hRb)
    _, ch, cR = backward(prob, u1, hh, hR, hs, hr, N, hRb)
    for got, ref in ((Yg.grad, aY + bY), (hg.grad, bh + ch), (Rg.grad, aR + cR), (Rbg.grad, dA_bar)):
        assert _rel(got.cpu(), ref) < TOL


def test_tp_graph_reuse_flag():
    """SYMCON_TP_REUSE_GRAPH (the backward of a step keeps the receiver / sender CSR its forward or an
    earlier backward built on the same workspace): outputs bitwise equal to the rebuild path, fewer
    launches; a different graph with the flag set (other pointers) is detected and rebuilt; the oracle
    still agrees on the second graph."""
    from oracle.tp import TPProblem, backward
    tp, Y, h, R, s, r, N = _setup(3, (0, 1), 3, 64, [30, 22, 41], seed=4)
    dA = torch.randn((N, 64, tp.n_out), generator=torch.Generator("cuda").manual_seed(2), device="cuda")
    tp.forward_raw(Y, h, R, s, r)
    ref = tp.backward_raw(Y, h, R, s, r, dA)                 # rebuilds everything
    n_full = tp.last_launch_count()
    tp.forward_raw(Y, h, R, s, r)
    got = tp.backward_raw(Y, h, R, s, r, dA, reuse=True)     # recv part from the forward
    n_reuse1 = tp.last_launch_count()
    got2 = tp.backward_raw(Y, h, R, s, r, dA, reuse=True)    # recv and sender CSR both kept
    n_reuse2 = tp.last_launch_count()
    torch.cuda.synchronize()
    assert tp.check_device_error()[0] == 0
    for a, b, c in zip(ref, got, got2):
        assert torch.equal(a, b) and torch.equal(a, c)
    assert n_reuse2 < n_reuse1 < n_full, (n_full, n_reuse1, n_reuse2)
    # SYMCON_TP_PREP_BACKWARD: the forward builds the sender CSR concurrently; the backward builds nothing
    A0 = tp.forward_raw(Y, h, R, s, r)
    A1 = tp.forward_raw(Y, h, R, s, r, prep_backward=True)
    got3 = tp.backward_raw(Y, h, R, s, r, dA, reuse=True)
    n_prep = tp.last_launch_count()
    torch.cuda.synchronize()
    assert torch.equal(A0, A1)
    for a, c in zip(ref, got3):
        assert torch.equal(a, c)
    assert n_prep == n_reuse2, (n_prep, n_reuse2)
    # another graph (new index tensors) with the flag: must not reuse the old structure
    from synth.inputs import gen_tp_graph
    sizes2 = [25, 47]
    s2, r2 = gen_tp_graph(sizes2, 30, 9)
    N2, E2 = int(sum(sizes2)), len(s2)
    s2, r2 = torch.from_numpy(s2).cuda(), torch.from_numpy(r2).cuda()
    Y2, h2, R2 = Y[:E2].contiguous(), h[:N2].contiguous(), R[:E2].contiguous()
    dA2 = dA[:N2].contiguous()
    dY2, dh2, dR2 = tp.backward_raw(Y2, h2, R2, s2, r2, dA2, reuse=True)
    torch.cuda.synchronize()
    assert tp.check_device_error()[0] == 0
    prob = TPProblem(3, (0, 1), 3)
    hY, hh, hR, hs, hr, hdA = _host(Y2, h2, R2, s2, r2, dA2)
    rY, rh, rR = backward(prob, hY, hh, hR, hs, hr, N2, hdA)
    assert _rel(dY2.cpu(), rY) < TOL and _rel(dh2.cpu(), rh) < TOL and _rel(dR2.cpu(), rR) < TOL

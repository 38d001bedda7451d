"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerance: max|err| <= 1e-4 * max|ref| per tensor (north_star); internal gate 1e-5 (DESIGN.md
§7: fp32 rounding measured <= 4e-6 of max|ref|, so an error near 1e-4 is a bug).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _sc(lmax, corr, outs, E, K):
    from paper_2504_10700_b200.ops import SymmetricContraction
    return SymmetricContraction(lmax, corr, outs, E, K, device=0)


def _inputs(sc, N, dist="uniform", seed=0):
    from synth.inputs import gen_A, gen_W, gen_node_elem, gen_dB
    A = gen_A(N, sc.channels, sc.n_lm, "cuda", seed)
    W = gen_W(sc.num_elements, sc.block_sizes(), sc.channels, "cuda", seed)
    ne = gen_node_elem(N, sc.num_elements, dist, "cuda", seed)
    dB = gen_dB(N, sc.out_dim, "cuda", seed)
    return A, W, ne, dB


def _rel(x, ref):
    ref = np.asarray(ref, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    scale = np.abs(ref).max()
    return np.abs(x - ref).max() / (scale if scale > 0 else 1.0)


def _run(sc, A, W, ne, dB):
    B = sc.forward_raw(A, W, ne)
    dA, dW = sc.backward_raw(A, W, ne, dB)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    assert s == 0, bad
    return B, dA, dW


def _host(*ts):
    return [t.detach().cpu().numpy() for t in ts]


def test_tiny_against_python_oracle():
    from oracle.contraction import Problem, forward, backward
    sc = _sc(3, 3, (0,), 3, 16)
    A, W, ne, dB = _inputs(sc, 32)
    B, dA, dW = _run(sc, A, W, ne, dB)
    prob = Problem(3, 3, (0,))
    hA, hW, hne, hdB = _host(A, W, ne, dB)
    Bref = forward(prob, hA, hW, hne)
    dAref, dWref = backward(prob, hA, hW, hne, hdB)
    assert _rel(B.cpu(), Bref) < TOL
    assert _rel(dA.cpu(), dAref) < TOL
    assert _rel(dW.cpu(), dWref) < TOL


@pytest.mark.parametrize("name,lmax,corr,outs,E,K,N,dist", [
    ("off_small_shape", 3, 3, (0,), 10, 96, 3000, "organic"),
    ("mp_shape", 3, 3, (0, 1), 89, 128, 3000, "zipf"),
    ("large_shape", 3, 3, (0, 1, 2), 89, 256, 700, "zipf"),
    ("ragged_K13", 3, 3, (0, 1), 5, 13, 777, "uniform"),
    ("lmax2", 2, 3, (0, 1), 4, 24, 500, "uniform"),
    ("lmax1", 1, 3, (0, 1), 3, 8, 300, "uniform"),
    ("corr1_all_L", 3, 1, (0, 1, 2, 3), 3, 16, 300, "uniform"),
    ("corr2", 3, 2, (0, 1), 3, 16, 300, "uniform"),
    ("out_1o_only", 3, 3, (1,), 7, 32, 500, "zipf"),
    ("scalars_only_lmax0", 0, 3, (0,), 3, 16, 300, "uniform"),
    ("single_channel_element", 3, 3, (0, 1), 1, 1, 200, "uniform"),
    ("odd_K255", 3, 3, (0,), 4, 255, 300, "uniform"),
    ("out_2e_3o_corr2", 3, 2, (2, 3), 3, 24, 300, "uniform"),
    ("out_0123_corr3", 2, 3, (0, 1, 2, 3), 3, 8, 200, "uniform"),
])
def test_against_c_oracle(name, lmax, corr, outs, E, K, N, dist):
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    sc = _sc(lmax, corr, outs, E, K)
    A, W, ne, dB = _inputs(sc, N, dist, seed=11)
    B, dA, dW = _run(sc, A, W, ne, dB)
    oc = OracleC(Problem(lmax, corr, outs))
    hA, hW, hne, hdB = _host(A, W, ne, dB)
    Bref = oc.forward(hA, hW, hne)
    dAref, dWref = oc.backward(hA, hW, hne, hdB)
    assert _rel(B.cpu(), Bref) < TOL, name
    assert _rel(dA.cpu(), dAref) < TOL, name
    assert _rel(dW.cpu(), dWref) < TOL, name


def test_corr1_is_linear_map_exactly():
    sc = _sc(3, 1, (0, 1, 2, 3), 3, 16)
    A, W, ne, dB = _inputs(sc, 200)
    B = sc.forward_raw(A, W, ne)
    N, K = A.shape[:2]
    off = 0
    for c, L in enumerate((0, 1, 2, 3)):
        blk = B[:, off:off + K * (2 * L + 1)].reshape(N, K, 2 * L + 1)
        expect = W[ne.long()][:, c, :].unsqueeze(-1) * A[:, :, L * L:(L + 1) ** 2]
        assert torch.equal(blk, expect)
        off += K * (2 * L + 1)


def test_empty_elements_get_zero_dW_and_edge_sizes():
    sc = _sc(3, 3, (0, 1), 6, 16)
    for N in (1, 63, 64, 65, 129):
        A, W, _, dB = _inputs(sc, N)
        ne = torch.full((N,), 4, dtype=torch.int32, device="cuda")
        ne[: N // 2] = 1
        _, _, dW = _run(sc, A, W, ne, dB)
        for z in (0, 2, 3, 5):
            assert torch.count_nonzero(dW[z]) == 0
    # N = 0: no launch, dW overwritten with zeros
    A = torch.zeros((0, 16, 16), device="cuda")
    W = torch.randn((6, sc.n_paths, 16), device="cuda")
    ne = torch.zeros((0,), dtype=torch.int32, device="cuda")
    dB = torch.zeros((0, sc.out_dim), device="cuda")
    B = sc.forward_raw(A, W, ne)
    dW = torch.full_like(W, 7.0)
    sc.backward_raw(A, W, ne, dB, need_dA=False, dW=dW)
    torch.cuda.synchronize()
    assert B.shape == (0, sc.out_dim) and torch.count_nonzero(dW) == 0


def test_bad_element_is_reported_and_nan():
    sc = _sc(3, 3, (0,), 3, 8)
    A, W, ne, dB = _inputs(sc, 100)
    ne[17] = 3
    ne[40] = -1
    B = sc.forward_raw(A, W, ne)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    from paper_2504_10700_b200 import _lib
    assert s == _lib.SYMCON_EELEMENT and bad == 17
    assert torch.isnan(B[17]).all() and torch.isnan(B[40]).all()
    good = torch.ones(100, dtype=torch.bool)
    good[[17, 40]] = False
    assert torch.isfinite(B[good.cuda()]).all()


def test_deterministic_bitwise():
    sc = _sc(3, 3, (0, 1), 89, 64)
    A, W, ne, dB = _inputs(sc, 5000, "zipf")
    r1 = _run(sc, A, W, ne, dB)
    r2 = _run(sc, A, W, ne, dB)
    for a, b in zip(r1, r2):
        assert torch.equal(a, b)


def test_identities_on_gpu_outputs():
    """Oracle-free checks on fp32 outputs: <W,dW> = <dB,B> and the Euler identity."""
    sc = _sc(3, 3, (0, 1), 89, 128)
    A, W, ne, dB = _inputs(sc, 4000, "zipf")
    B, dA, dW = _run(sc, A, W, ne, dB)
    lhs = (W.double() * dW.double()).sum().item()
    rhs = (dB.double() * B.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-5 * (dB.double().abs() * B.double().abs()).sum().item()
    # Euler: sum_a A_a dA_a = sum_nu nu <dB, B_nu>; build B_nu by masking W columns
    e = (A.double() * dA.double()).sum()
    r = 0.0
    for nu in (1, 2, 3):
        Wn = W.clone()
        col = 0
        for (L, n, cnt) in sc.block_sizes():
            if n != nu:
                Wn[:, col:col + cnt] = 0
            col += cnt
        Bn = sc.forward_raw(A, Wn, ne)
        r += nu * (dB.double() * Bn.double()).sum()
    torch.cuda.synchronize()
    assert abs(e - r).item() <= 1e-5 * abs(r).item() + 1e-3


def test_full_size_mp_sampled():
    """MP-medium at full size (N=50k, the bench launch config): sampled nodes vs the oracle for
    B and dA; dW checked exactly on the three smallest elements (all their nodes)."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    from synth.inputs import CONFIGS
    cfg = CONFIGS["mp_medium"]
    sc = _sc(3, 3, cfg.out_L, cfg.n_elements, cfg.channels)
    A, W, ne, dB = _inputs(sc, cfg.n_nodes, cfg.elem_dist, seed=0)
    B, dA, dW = _run(sc, A, W, ne, dB)
    oc = OracleC(Problem(3, 3, cfg.out_L))
    rng = np.random.default_rng(123)
    idx = torch.tensor(np.sort(rng.choice(cfg.n_nodes, 96, replace=False)), device="cuda")
    hA, hW, hne, hdB = _host(A[idx], W, ne[idx], dB[idx])
    assert _rel(B[idx].cpu(), oc.forward(hA, hW, hne)) < TOL
    dAref, _ = oc.backward(hA, hW, hne, hdB, want_dW=False)
    assert _rel(dA[idx].cpu(), dAref) < TOL
    counts = torch.bincount(ne.long(), minlength=cfg.n_elements).cpu().numpy()
    for z in np.argsort(counts)[:3]:
        sel = torch.nonzero(ne == int(z)).flatten()
        hA, hne, hdB = _host(A[sel], ne[sel], dB[sel])
        _, dWref = oc.backward(hA, W.cpu().numpy(), hne, hdB, want_dA=False)
        assert _rel(dW[z].cpu(), dWref[z]) < TOL


def test_autograd_wrapper():
    sc = _sc(3, 3, (0, 1), 4, 16)
    A, W, ne, dB = _inputs(sc, 300)
    A.requires_grad_(True)
    W.requires_grad_(True)
    B = sc(A, W, ne)
    (B * dB).sum().backward()
    dA, dW = sc.backward_raw(A.detach(), W.detach(), ne, dB)
    torch.cuda.synchronize()
    assert torch.equal(A.grad, dA) and torch.equal(W.grad, dW)


def test_reuse_hints_never_change_results():
    sc = _sc(3, 3, (0, 1), 7, 32)
    A, W, ne, dB = _inputs(sc, 900, "zipf")
    ref_dA, ref_dW = sc.backward_raw(A, W, ne, dB)
    sc.forward_raw(A, W, ne)
    dA1, dW1 = sc.backward_raw(A, W, ne, dB, reuse=True)          # reuses buckets + fold
    ne2 = ne.flip(0).contiguous()                                   # different pointer and contents
    sc.forward_raw(A, W, ne2)
    dA2, dW2 = sc.backward_raw(A, W, ne, dB, reuse=True)           # hint must not apply: redone
    W2 = (W * 2).contiguous()
    sc.forward_raw(A, W2, ne)
    dA3, _ = sc.backward_raw(A, W, ne, dB, reuse=True)             # same ne, other W: fold redone
    torch.cuda.synchronize()
    for x, y in ((dA1, ref_dA), (dW1, ref_dW), (dA2, ref_dA), (dW2, ref_dW), (dA3, ref_dA)):
        assert torch.equal(x, y)


def test_full_size_off_small_all_nodes():
    """OFF-small at full size (20k nodes of 10-100-atom molecules, 96 channels, 0e): every output
    element against the C oracle."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    from synth.inputs import CONFIGS, make_config_inputs
    cfg = CONFIGS["off_small"]
    sc = _sc(3, 3, cfg.out_L, cfg.n_elements, cfg.channels)
    A, W, ne, dB = make_config_inputs(cfg, sc.block_sizes(), sc.out_dim, device="cuda")
    B, dA, dW = _run(sc, A, W, ne, dB)
    oc = OracleC(Problem(3, 3, cfg.out_L))
    hA, hW, hne, hdB = _host(A, W, ne, dB)
    assert _rel(B.cpu(), oc.forward(hA, hW, hne)) < TOL
    dAref, dWref = oc.backward(hA, hW, hne, hdB)
    assert _rel(dA.cpu(), dAref) < TOL
    assert _rel(dW.cpu(), dWref) < TOL


def test_full_size_large_sampled():
    """Large (200k nodes, 256 channels, 0e+1o+2e): sampled nodes for B and dA, dW exactly on the
    two smallest elements."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    from synth.inputs import CONFIGS, make_config_inputs
    cfg = CONFIGS["large"]
    sc = _sc(3, 3, cfg.out_L, cfg.n_elements, cfg.channels)
    A, W, ne, dB = make_config_inputs(cfg, sc.block_sizes(), sc.out_dim, device="cuda")
    B, dA, dW = _run(sc, A, W, ne, dB)
    oc = OracleC(Problem(3, 3, cfg.out_L))
    rng = np.random.default_rng(7)
    idx = torch.tensor(np.sort(rng.choice(cfg.n_nodes, 48, replace=False)), device="cuda")
    hA, hW, hne, hdB = _host(A[idx], W, ne[idx], dB[idx])
    assert _rel(B[idx].cpu(), oc.forward(hA, hW, hne)) < TOL
    dAref, _ = oc.backward(hA, hW, hne, hdB, want_dW=False)
    assert _rel(dA[idx].cpu(), dAref) < TOL
    counts = torch.bincount(ne.long(), minlength=cfg.n_elements).cpu().numpy()
    for z in np.argsort(counts)[:2]:
        sel = torch.nonzero(ne == int(z)).flatten()
        hA, hne, hdB = _host(A[sel], ne[sel], dB[sel])
        _, dWref = oc.backward(hA, hW, hne, hdB, want_dA=False)
        assert _rel(dW[z].cpu(), dWref[z]) < TOL
    del A, dB, B, dA
    torch.cuda.empty_cache()


def test_sharded_dp_step_matches_single_pass():
    """Data-parallel plumbing on one GPU: the dW of two bins computed separately and summed equals
    the dW of their union (what the NCCL all-reduce produces across ranks), bitwise up to the
    fp32 sum order tolerance."""
    from synth.inputs import table2_sizes, graph_elements
    from paper_2504_10700_b200.dist import BinPackedShards
    sc = _sc(3, 3, (0, 1), 89, 64)
    sizes = table2_sizes(scale=0.002)
    sh = BinPackedShards(sizes, 3072, 2, 0)
    parts = []
    for r in range(2):
        g = sh.graphs(0, r)
        ne = torch.from_numpy(graph_elements(sizes[g], salt=r)).cuda()
        A = torch.randn((ne.numel(), 64, 16), device="cuda")
        dB = torch.randn((ne.numel(), sc.out_dim), device="cuda")
        parts.append((A, ne, dB))
    from synth.inputs import gen_W
    W = gen_W(89, sc.block_sizes(), 64, "cuda")
    dWs = [sc.backward_raw(A, W, ne, dB, need_dA=False)[1].clone() for A, ne, dB in parts]
    Au = torch.cat([p[0] for p in parts]).contiguous()
    neu = torch.cat([p[1] for p in parts]).contiguous()
    dBu = torch.cat([p[2] for p in parts]).contiguous()
    _, dWu = sc.backward_raw(Au, W, neu, dBu, need_dA=False)
    torch.cuda.synchronize()
    s = dWs[0] + dWs[1]
    assert (s - dWu).abs().max().item() <= 1e-5 * dWu.abs().max().item()


# ---------------------------------------------------------------- double backward (§8(f) row 1)
def _uA(sc, N, seed):
    from synth.inputs import gen_A
    return gen_A(N, sc.channels, sc.n_lm, "cuda", seed + 1000)


def test_backward2_tiny_against_python_oracle():
    from oracle.contraction import Problem, backward2
    sc = _sc(3, 3, (0, 1), 3, 16)
    A, W, ne, dB = _inputs(sc, 70)
    uA = _uA(sc, 70, 0)
    got = sc.backward2_raw(A, W, ne, dB, uA)
    torch.cuda.synchronize()
    ref = backward2(Problem(3, 3, (0, 1)), *_host(A, W, ne, dB, uA))
    for g, r in zip(got, ref):
        assert _rel(g.cpu(), r) < TOL


@pytest.mark.parametrize("name,lmax,corr,outs,E,K,N,dist", [
    ("off_small_shape", 3, 3, (0,), 10, 96, 2000, "organic"),
    ("mp_shape", 3, 3, (0, 1), 89, 128, 2000, "zipf"),
    ("large_shape", 3, 3, (0, 1, 2), 89, 256, 400, "zipf"),
    ("ragged_K13", 3, 3, (0, 1), 5, 13, 777, "uniform"),
    ("lmax2", 2, 3, (0, 1), 4, 24, 500, "uniform"),
    ("corr1_all_L", 3, 1, (0, 1, 2, 3), 3, 16, 300, "uniform"),
    ("corr2", 3, 2, (0, 1), 3, 16, 300, "uniform"),
    ("out_1o_only", 3, 3, (1,), 7, 32, 500, "zipf"),
    ("scalars_only_lmax0", 0, 3, (0,), 3, 16, 300, "uniform"),
    ("odd_K255", 3, 3, (0,), 4, 255, 200, "uniform"),
    ("out_2e_3o_corr2", 3, 2, (2, 3), 3, 24, 300, "uniform"),
])
def test_backward2_against_c_oracle(name, lmax, corr, outs, E, K, N, dist):
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    sc = _sc(lmax, corr, outs, E, K)
    A, W, ne, dB = _inputs(sc, N, dist, seed=5)
    uA = _uA(sc, N, 5)
    got = sc.backward2_raw(A, W, ne, dB, uA)
    torch.cuda.synchronize()
    assert sc.check_device_error()[0] == 0
    ref = OracleC(Problem(lmax, corr, outs)).backward2(*_host(A, W, ne, dB, uA))
    for what, g, r in zip(("dB_bar", "A_bar", "W_bar"), got, ref):
        if np.abs(r).max() == 0:          # corr1: the map is linear in A, A_bar = 0 exactly
            assert torch.count_nonzero(g) == 0, (name, what)
        else:
            assert _rel(g.cpu(), r) < TOL, (name, what)


def test_backward2_subsets_edges_and_bad_elements():
    from paper_2504_10700_b200 import _lib
    sc = _sc(3, 3, (0, 1), 6, 16)
    A, W, ne, dB = _inputs(sc, 129)
    uA = _uA(sc, 129, 0)
    full = sc.backward2_raw(A, W, ne, dB, uA)
    for mask in ((True, False, False), (False, True, False), (False, False, True)):
        part = sc.backward2_raw(A, W, ne, dB, uA, *mask)
        for m, f, p in zip(mask, full, part):
            assert (p is None) != m and (p is None or torch.equal(p, f))
    # elements without nodes: W_bar = 0; N = 0 overwrites W_bar with zeros
    ne2 = torch.full_like(ne, 4)
    _, _, Wb = sc.backward2_raw(A, W, ne2, dB, uA)
    for z in (0, 1, 2, 3, 5):
        assert torch.count_nonzero(Wb[z]) == 0
    e = lambda *s: torch.zeros(s, device="cuda")
    _, _, Wb = sc.backward2_raw(e(0, 16, 16), W, torch.zeros(0, dtype=torch.int32, device="cuda"),
                                e(0, sc.out_dim), e(0, 16, 16), need_dB=False, need_A=False)
    torch.cuda.synchronize()
    assert torch.count_nonzero(Wb) == 0
    # an out-of-range element: NaN rows and SYMCON_EELEMENT, like the forward
    ne3 = ne.clone()
    ne3[33] = 6
    dBb, Ab, _ = sc.backward2_raw(A, W, ne3, dB, uA)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    assert s == _lib.SYMCON_EELEMENT and bad == 33
    assert torch.isnan(dBb[33]).all() and torch.isnan(Ab[33]).all()
    ok = torch.ones(129, dtype=torch.bool, device="cuda")
    ok[33] = False
    assert torch.isfinite(dBb[ok]).all() and torch.isfinite(Ab[ok]).all()


def test_double_backward_autograd_force_loss():
    """Training on forces: E = <R, B(A, W)>, F-like term dA = dE/dA with create_graph=True, loss
    <V, dA> + <VW, dW>; its gradients against the oracle (uA terms: backward2; uW terms: the
    forward and the dA backward with W -> VW, ops._SymconBwdFn)."""
    from oracle.contraction import Problem, backward, backward2, forward
    sc = _sc(3, 3, (0, 1), 4, 16)
    A0, W0, ne, R0 = _inputs(sc, 90)
    V = _uA(sc, 90, 0)
    VW = torch.randn(W0.shape, generator=torch.Generator("cuda").manual_seed(3), device="cuda")
    A, W, R = (x.clone().requires_grad_(True) for x in (A0, W0, R0))
    E = (sc(A, W, ne) * R).sum()
    dA, dW = torch.autograd.grad(E, (A, W), create_graph=True)
    loss = (dA * V).sum() + (dW * VW).sum()
    loss.backward()
    prob = Problem(3, 3, (0, 1))
    hA, hW, hne, hR, hV, hVW = _host(A0, W0, ne, R0, V, VW)
    dBb, Ab, Wb = backward2(prob, hA, hW, hne, hR, hV)
    Ab = Ab + backward(prob, hA, hVW, hne, hR)[0]
    dBb = dBb + forward(prob, hA, hVW, hne)
    assert _rel(A.grad.cpu(), Ab) < TOL
    assert _rel(W.grad.cpu(), Wb) < TOL
    assert _rel(R.grad.cpu(), dBb) < TOL


@pytest.mark.parametrize("config", ["mp_medium", "large"])
def test_backward2_full_size_sampled(config):
    """Double backward at full size: sampled nodes vs the oracle for dB_bar and A_bar (each
    depends on its own node only); W_bar exactly on the three smallest elements (all their
    nodes) and, over all elements, the bilinear identity <W, W_bar> = <dB, dB_bar>."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    from synth.inputs import CONFIGS
    cfg = CONFIGS[config]
    n = cfg.n_nodes if config == "mp_medium" else 60000
    sc = _sc(3, 3, cfg.out_L, cfg.n_elements, cfg.channels)
    A, W, ne, dB = _inputs(sc, n, cfg.elem_dist, seed=1)
    uA = _uA(sc, n, 1)
    dBb, Ab, Wb = sc.backward2_raw(A, W, ne, dB, uA)
    torch.cuda.synchronize()
    assert sc.check_device_error()[0] == 0
    oc = OracleC(Problem(3, 3, cfg.out_L))
    rng = np.random.default_rng(7)
    idx = torch.tensor(np.sort(rng.choice(n, 48, replace=False)), device="cuda")
    ref = oc.backward2(*_host(A[idx], W, ne[idx], dB[idx], uA[idx]), want_W=False)
    assert _rel(dBb[idx].cpu(), ref[0]) < TOL
    assert _rel(Ab[idx].cpu(), ref[1]) < TOL
    counts = torch.bincount(ne.long(), minlength=cfg.n_elements).cpu().numpy()
    for z in np.argsort(counts)[:3]:
        sel = torch.nonzero(ne == int(z)).flatten()
        if sel.numel() == 0:
            assert torch.count_nonzero(Wb[z]) == 0
            continue
        _, _, Wref = oc.backward2(*_host(A[sel], W, ne[sel], dB[sel], uA[sel]), want_dB=False, want_A=False)
        assert _rel(Wb[z].cpu(), Wref[z]) < TOL
    lhs = (W.double() * Wb.double()).sum().item()
    rhs = (dB.double() * dBb.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-5 * (W.double().abs() * Wb.double().abs()).sum().item()
    del A, dB, uA, dBb, Ab
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,lmax,corr,outs,E,K,N,with_uA", [
    ("mp_shape_uW_only", 3, 3, (0, 1), 89, 128, 2000, False),
    ("mp_shape_uA_uW", 3, 3, (0, 1), 89, 128, 2000, True),
    ("off_shape_uA_uW", 3, 3, (0,), 10, 96, 1500, True),
    ("large_shape_uW_only", 3, 3, (0, 1, 2), 89, 256, 400, False),
])
def test_backward2_ex_uW_terms_in_library(name, lmax, corr, outs, E, K, N, with_uA):
    """symcon_backward2_ex: the cotangent uW of dW adds dB_bar += forward(A, uW) and A_bar += dA(A, uW, dB)
    inside libsymcon (second fold + accumulating forward / dA kernels), no caller arithmetic."""
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    sc = _sc(lmax, corr, outs, E, K)
    A, W, ne, dB = _inputs(sc, N, "zipf", seed=5)
    uA = _uA(sc, N, 5) if with_uA else None
    uW = torch.randn(W.shape, generator=torch.Generator("cuda").manual_seed(8), device="cuda")
    dBb, Ab, Wb = sc.backward2_raw(A, W, ne, dB, uA, uW=uW)
    torch.cuda.synchronize()
    assert sc.check_device_error()[0] == 0
    oc = OracleC(Problem(lmax, corr, outs))
    hA, hW, hne, hdB, huW = _host(A, W, ne, dB, uW)
    dB_ref = oc.forward(hA, huW, hne)
    A_ref = oc.backward(hA, huW, hne, hdB, want_dW=False)[0]
    if with_uA:
        r = oc.backward2(hA, hW, hne, hdB, uA.cpu().numpy())
        dB_ref, A_ref = dB_ref + r[0], A_ref + r[1]
        assert _rel(Wb.cpu(), r[2]) < TOL
    else:
        assert torch.count_nonzero(Wb) == 0
    assert _rel(dBb.cpu(), dB_ref) < TOL, name
    assert _rel(Ab.cpu(), A_ref) < TOL, name

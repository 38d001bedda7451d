"""Interaction + product block chained through autograd on the GPU (SURVEY §8(f) rows 1-2 with
§8(a)): channelwise TP (Alg. 2 + neighbour sum) -> A -> symmetric contraction -> B, loss <B, Rb>,
gradients w.r.t. Y, h, R (TP inputs) and W (contraction weights) against the chained fp64 oracle."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_tp_then_contraction_autograd_chain():
    from paper_2504_10700_b200.ops import ChannelwiseTP, SymmetricContraction
    from synth.inputs import gen_tp_graph, gen_tp_inputs, gen_W, gen_node_elem
    from oracle import tp as otp
    from oracle.contraction import Problem, forward as cforward, backward as cbackward
    K, E_el = 32, 5
    tp = ChannelwiseTP(3, (0, 1), 3, K, device=0)
    sc = SymmetricContraction(3, 3, (0, 1), E_el, K, device=0)
    s_np, r_np = gen_tp_graph([11, 17, 9], 6, seed=2)
    N, E = 37, len(s_np)
    Y, h, R = gen_tp_inputs(N, E, K, tp.n_y, tp.n_h, tp.n_paths, "cuda", seed=2)
    Y, h, R = (x * 0.3 for x in (Y, h, R))   # keep the cubic contraction of the summed messages O(1)
    W = gen_W(E_el, sc.block_sizes(), K, "cuda", seed=2)
    ne = gen_node_elem(N, E_el, "uniform", "cuda", seed=2)
    s, r = torch.from_numpy(s_np).cuda(), torch.from_numpy(r_np).cuda()
    Rb = torch.randn((N, sc.out_dim), generator=torch.Generator("cuda").manual_seed(4), device="cuda")
    Yg, hg, Rg, Wg = (x.clone().contiguous().requires_grad_(True) for x in (Y, h, R, W))
    A = tp(Yg, hg, Rg, s, r)
    B = sc(A, Wg, ne)
    (B * Rb).sum().backward()
    torch.cuda.synchronize()
    # oracle chain
    hY, hh, hR, hW, hne, hRb = (x.detach().cpu().numpy() for x in (Y, h, R, W, ne, Rb))
    tprob, cprob = otp.TPProblem(3, (0, 1), 3), Problem(3, 3, (0, 1))
    Aref = otp.forward(tprob, hY, hh, hR, s_np, r_np, N)
    Bref = cforward(cprob, Aref, hW, hne)
    dAref, dWref = cbackward(cprob, Aref, hW, hne, hRb)
    dYref, dhref, dRref = otp.backward(tprob, hY, hh, hR, s_np, r_np, N, dAref)

    def rel(x, ref):
        return np.abs(x.detach().cpu().numpy().astype(np.float64) - ref).max() / np.abs(ref).max()
    # fp32 end to end through two cubic/bilinear stages: gate 1e-4 (north_star bound)
    for name, x, ref in (("A", A, Aref), ("B", B, Bref), ("dW", Wg.grad, dWref), ("dY", Yg.grad, dYref),
                         ("dh", hg.grad, dhref), ("dR", Rg.grad, dRref)):
        assert rel(x, ref) < 1e-4, name


def test_force_style_loss_through_tp_and_contraction():
    """create_graph=True through both blocks: E = <B(A(Y, h, R), W), Rb>, loss = <dE/dY, V>; the
    gradients w.r.t. Y and W against the oracle chain (TP forward with Y := V, the contraction's
    double backward with uA = that, the TP backward of the result)."""
    from paper_2504_10700_b200.ops import ChannelwiseTP, SymmetricContraction
    from synth.inputs import gen_tp_graph, gen_tp_inputs, gen_W, gen_node_elem
    from oracle import tp as otp
    from oracle.contraction import Problem, backward2 as cbackward2
    K, E_el = 32, 4
    tp = ChannelwiseTP(3, (0, 1), 3, K, device=0)
    sc = SymmetricContraction(3, 3, (0, 1), E_el, K, device=0)
    s_np, r_np = gen_tp_graph([10, 14], 5, seed=3)
    N, E = 24, len(s_np)
    Y, h, R = (x * 0.3 for x in gen_tp_inputs(N, E, K, tp.n_y, tp.n_h, tp.n_paths, "cuda", seed=3))
    W = gen_W(E_el, sc.block_sizes(), K, "cuda", seed=3)
    ne = gen_node_elem(N, E_el, "uniform", "cuda", seed=3)
    s, r = torch.from_numpy(s_np).cuda(), torch.from_numpy(r_np).cuda()
    g = torch.Generator("cuda").manual_seed(8)
    Rb = torch.randn((N, sc.out_dim), generator=g, device="cuda")
    V = torch.randn(Y.shape, generator=g, device="cuda")
    Yg, Wg = Y.clone().contiguous().requires_grad_(True), W.clone().contiguous().requires_grad_(True)
    Ecal = (sc(tp(Yg, h, R, s, r), Wg, ne) * Rb).sum()
    (gY,) = torch.autograd.grad(Ecal, (Yg,), create_graph=True)
    (gY * V).sum().backward()
    torch.cuda.synchronize()
    hY, hh, hR, hW, hne, hRb, hV = (x.detach().cpu().numpy() for x in (Y, h, R, W, ne, Rb, V))
    tprob, cprob = otp.TPProblem(3, (0, 1), 3), Problem(3, 3, (0, 1))
    A = otp.forward(tprob, hY, hh, hR, s_np, r_np, N)
    uA = otp.forward(tprob, hV, hh, hR, s_np, r_np, N)                  # dA_bar of the TP double backward
    _, A_bar, W_bar = cbackward2(cprob, A, hW, hne, hRb, uA)
    Y_ref = otp.backward(tprob, hY, hh, hR, s_np, r_np, N, A_bar)[0]

    def rel(x, ref):
        return np.abs(x.detach().cpu().numpy().astype(np.float64) - ref).max() / np.abs(ref).max()
    assert rel(Yg.grad, Y_ref) < 1e-4
    assert rel(Wg.grad, W_bar) < 1e-4

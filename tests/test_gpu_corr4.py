"""Correlation 4 ("all possible combinations ... that would
result in a nonzero contribution" at nu = 4; reading s4b): the plain scalar kernels of
codegen_simple.cpp (prefix-trie forward, reverse-mode dA, S-route dW) through the C ABI, against the
plain C fp64 oracle (oracle/csrc/oracle_eval.c, pinned in tests/test_oracle_corr4.py) on the same
seeded inputs, element by element.

Tolerances: fp32 max|err| <= 1e-5 * max|ref| per tensor (the internal gate; north_star 1e-4): the
degree-4 products add one rounding per term over corr 3 (~1e-7 relative each) and the dW sums run over
up to ~1e3 nodes of one element; fp64 1e-10 * max|ref| (test_gpu_f64.py's bar).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL32, TOL64 = 1e-5, 1e-10


def _rel(x, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.abs(np.asarray(x, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-300))


@pytest.mark.parametrize("name,lmax,outs,E,K,N,dist,dtype", [
    ("mp_shape_f32", 3, (0, 1), 10, 128, 600, "zipf", torch.float32),
    ("off_shape_f32", 3, (0,), 6, 96, 300, "organic", torch.float32),
    ("ragged_K13_f32", 3, (0, 1), 3, 13, 130, "uniform", torch.float32),
    ("lmax2_three_outs_f32", 2, (0, 1, 2), 4, 32, 200, "uniform", torch.float32),
    ("off_shape_f64", 3, (0,), 5, 64, 150, "zipf", torch.float64),
    ("lmax2_f64", 2, (0, 1), 4, 40, 170, "uniform", torch.float64),
])
def test_corr4_against_c_oracle(name, lmax, outs, E, K, N, dist, dtype):
    from paper_2504_10700_b200.ops import SymmetricContraction
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    from synth.inputs import gen_A, gen_W, gen_node_elem, gen_dB
    sc = SymmetricContraction(lmax, 4, outs, E, K, device=0, dtype=dtype)
    assert sc.info.correlation == 4
    A = gen_A(N, K, sc.n_lm, "cpu", 5).to(dtype).cuda()
    W = gen_W(E, sc.block_sizes(), K, "cpu", 5).to(dtype).cuda()
    ne = gen_node_elem(N, E, dist, "cuda", 5)
    dB = gen_dB(N, sc.out_dim, "cpu", 5).to(dtype).cuda()
    B = sc.forward_raw(A, W, ne)
    dA, dW = sc.backward_raw(A, W, ne, dB)
    torch.cuda.synchronize()
    assert sc.check_device_error()[0] == 0
    oc = OracleC(Problem(lmax, 4, outs))
    hA, hW, hne, hdB = (t.cpu().double().numpy() for t in (A, W, ne, dB))
    hne = ne.cpu().numpy()
    Bref = oc.forward(hA, hW, hne)
    dAref, dWref = oc.backward(hA, hW, hne, hdB)
    tol = TOL64 if dtype == torch.float64 else TOL32
    eB, eA, eW = _rel(B.cpu(), Bref), _rel(dA.cpu(), dAref), _rel(dW.cpu(), dWref)
    assert eB < tol and eA < tol and eW < tol, (name, eB, eA, eW)


def test_corr4_autograd_and_refusals():
    """torch.autograd through the corr-4 plan (first derivatives) matches the raw calls; the double
    backward is refused (symcon_backward2 is correlation <= 3 only); N = 0 zeroes dW."""
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200 import _lib
    sc = SymmetricContraction(3, 4, (0, 1), 3, 32, device=0)
    g = torch.Generator().manual_seed(3)
    A = torch.randn(40, 32, 16, generator=g).cuda().requires_grad_()
    W = torch.randn(3, sc.n_paths, 32, generator=g).cuda().requires_grad_()
    ne = (torch.arange(40) % 3).int().cuda()
    B = sc(A, W, ne)
    dB = torch.randn(B.shape, generator=g).cuda()
    (B * dB).sum().backward()
    dA, dW = sc.backward_raw(A.detach(), W.detach(), ne, dB)
    torch.cuda.synchronize()
    assert torch.equal(A.grad, dA) and torch.equal(W.grad, dW)
    ws = sc.workspace(40)
    with pytest.raises(_lib.SymconError):
        _lib.symcon_backward2(sc.plan, 40, A.data_ptr(), W.data_ptr(), ne.data_ptr(), dB.data_ptr(), A.data_ptr(),
                              None, None, W.data_ptr(), ws.data_ptr(), ws.numel(), 0, torch.cuda.current_stream().cuda_stream)
    _, dW0 = sc.backward_raw(A.detach()[:0], W.detach(), ne[:0], dB[:0])
    torch.cuda.synchronize()
    assert torch.count_nonzero(dW0) == 0

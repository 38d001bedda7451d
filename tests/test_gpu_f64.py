"""fp64 mode (the paper's Float64 runs): the fp64 plan
(symcon_build_tables_ex(..., SYMCON_F64), symcon_forward_f64 / symcon_backward_f64) against the fp64
Python oracle on the same float64 inputs, element by element.

Tolerance: max|err| <= 1e-10 * max|ref| per tensor. Both sides evaluate the same exact sums in fp64;
only the summation order differs (folded sorted monomials vs raw ordered tuples), so the expected
relative error is a few 1e-15 (terms ~ O(1), up to ~1e4 of them in the largest dW sums); 1e-10 leaves
five orders of headroom and still fails any indexing or coefficient error.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL64 = 1e-10


def _rel(x, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.abs(np.asarray(x, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-300))


@pytest.mark.parametrize("name,lmax,corr,outs,E,K,N,dist", [
    ("tiny", 3, 3, (0,), 3, 16, 32, "uniform"),
    ("off_shape", 3, 3, (0,), 10, 96, 150, "organic"),
    ("mp_shape", 3, 3, (0, 1), 89, 128, 200, "zipf"),
    ("large_shape", 3, 3, (0, 1, 2), 9, 64, 80, "zipf"),
    ("corr2_lmax2", 2, 2, (0, 1), 4, 24, 100, "uniform"),
    ("ragged_K13", 3, 3, (0, 1), 5, 13, 130, "uniform"),
])
def test_f64_against_python_oracle(name, lmax, corr, outs, E, K, N, dist):
    from paper_2504_10700_b200.ops import SymmetricContraction
    from oracle.contraction import Problem, forward, backward
    from synth.inputs import gen_A, gen_W, gen_node_elem, gen_dB
    sc = SymmetricContraction(lmax, corr, outs, E, K, device=0, dtype=torch.float64)
    assert sc.info.reserved == 1   # SYMCON_F64
    A = gen_A(N, K, sc.n_lm, "cpu", 3).double().cuda()
    W = gen_W(E, sc.block_sizes(), K, "cpu", 3).double().cuda()
    ne = gen_node_elem(N, E, dist, "cuda", 3)
    dB = gen_dB(N, sc.out_dim, "cpu", 3).double().cuda()
    B = sc.forward_raw(A, W, ne)
    dA, dW = sc.backward_raw(A, W, ne, dB)
    torch.cuda.synchronize()
    assert sc.check_device_error()[0] == 0
    assert B.dtype == dA.dtype == dW.dtype == torch.float64
    prob = Problem(lmax, corr, outs)
    hA, hW, hne, hdB = (t.cpu().numpy() for t in (A, W, ne, dB))
    Bref = forward(prob, hA, hW, hne)
    dAref, dWref = backward(prob, hA, hW, hne, hdB)
    eB, eA, eW = _rel(B.cpu(), Bref), _rel(dA.cpu(), dAref), _rel(dW.cpu(), dWref)
    assert eB < TOL64 and eA < TOL64 and eW < TOL64, (name, eB, eA, eW)


def test_f64_dtype_mismatch_and_empty():
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200 import _lib
    sc = SymmetricContraction(3, 3, (0, 1), 4, 32, device=0, dtype=torch.float64)
    A = torch.randn(10, 32, 16, device="cuda", dtype=torch.float64)
    W = torch.randn(4, sc.n_paths, 32, device="cuda", dtype=torch.float64)
    ne = torch.zeros(10, dtype=torch.int32, device="cuda")
    ws = sc.workspace(10)
    B = torch.empty((10, sc.out_dim), device="cuda", dtype=torch.float64)
    with pytest.raises(_lib.SymconError):   # the fp32 entry point refuses an fp64 plan
        _lib.symcon_forward(sc.plan, 10, A.data_ptr(), W.data_ptr(), ne.data_ptr(), B.data_ptr(), ws.data_ptr(),
                            ws.numel(), torch.cuda.current_stream().cuda_stream)
    with pytest.raises(_lib.SymconError):   # double backward is fp32 only
        _lib.symcon_backward2(sc.plan, 10, A.data_ptr(), W.data_ptr(), ne.data_ptr(), B.data_ptr(), A.data_ptr(),
                              None, None, W.data_ptr(), ws.data_ptr(), ws.numel(), 0, torch.cuda.current_stream().cuda_stream)
    # N = 0: dW overwritten with exact zeros; element without nodes: dW = 0
    _, dW = sc.backward_raw(A[:0], W, ne[:0], torch.empty((0, sc.out_dim), device="cuda", dtype=torch.float64))
    torch.cuda.synchronize()
    assert torch.count_nonzero(dW) == 0
    dB = torch.randn((10, sc.out_dim), device="cuda", dtype=torch.float64)
    _, dW = sc.backward_raw(A, W, ne, dB)
    torch.cuda.synchronize()
    assert torch.count_nonzero(dW[1:]) == 0 and torch.count_nonzero(dW[0]) > 0

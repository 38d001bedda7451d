"""CPU checks of the C-ABI library: loads, exports every symbol of include/symcon.h, builds
host tables identical to the oracle's, and the host partitioner equals the oracle's Alg. 1."""
import os
import re
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2504_10700_b200 import build_lib
    build_lib.build()
    from paper_2504_10700_b200 import _lib
    return _lib


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "symcon.h")).read()
    names = set(re.findall(r"\b(symcon_[a-z0-9_]+)\s*\(", hdr))
    assert {"symcon_build_tables", "symcon_forward", "symcon_backward"} <= names
    for n in sorted(names):
        assert hasattr(L.lib, n), n


def test_invalid_arguments(L):
    with pytest.raises(L.SymconError) as e:
        L.symcon_build_tables(3, 5, [0], 2, 8, -1)
    assert e.value.status == L.SYMCON_EUNSUPPORTED
    plan4 = L.symcon_build_tables(3, 4, [0], 2, 8, -1)   # correlation 4: mono3 export refused
    with pytest.raises(L.SymconError) as e:
        L.symcon_plan_sym_table(plan4)
    assert e.value.status == L.SYMCON_EUNSUPPORTED
    L.symcon_destroy(plan4)
    for args in [(4, 3, [0]), (3, 0, [0]), (3, 3, [1, 0]), (3, 3, [])]:
        with pytest.raises(L.SymconError) as e:
            L.symcon_build_tables(args[0], args[1], args[2], 2, 8, -1)
        assert e.value.status == L.SYMCON_EINVAL
    plan = L.symcon_build_tables(3, 3, [0], 2, 8, -1)
    with pytest.raises(L.SymconError):   # host-only plan cannot compute
        L.symcon_forward(plan, 4, 16, 16, 16, 16, 16, 1 << 20, None)
    with pytest.raises(L.SymconError):
        L.symcon_backward2(plan, 4, 16, 16, 16, 16, 16, 16, 16, 16, 16, 1 << 20, 0, None)
    L.symcon_destroy(plan)


def test_real_cg_parity_with_oracle(L):
    from oracle.so3 import real_cg
    for l1 in range(4):
        for l2 in range(4):
            for J in range(abs(l1 - l2), min(6, l1 + l2) + 1):
                assert np.abs(L.symcon_real_cg(l1, l2, J) - real_cg(l1, l2, J)).max() < 1e-12


@pytest.mark.parametrize("lmax,corr,outs", [(3, 3, (0,)), (3, 3, (0, 1)), (3, 3, (0, 1, 2)), (2, 3, (0, 1)),
                                            (3, 1, (0, 1, 2, 3)), (3, 2, (1,)), (3, 4, (0, 1)), (2, 4, (0, 1, 2))])
def test_tables_parity_with_oracle(L, lmax, corr, outs):
    from oracle.contraction import Problem
    plan = L.symcon_build_tables(lmax, corr, list(outs), 3, 8, -1)
    info = L.symcon_plan_info(plan)
    prob = Problem(lmax, corr, outs)
    assert info.n_paths == prob.n_paths
    assert info.n_raw_terms == sum(len(p.terms) for p in prob.paths)
    for c, p in enumerate(prob.paths):
        assert L.symcon_plan_path(plan, c) == (p.L, p.nu, p.eta, p.ls, p.mids)
    acc = {}
    W = 4 if corr == 4 else 3
    for p in prob.paths:
        for M, ts, u in p.terms:
            key = (p.L, M, tuple(sorted(ts)) + (-1,) * (W - len(ts)), p.col)
            acc[key] = acc.get(key, 0.0) + u
    acc = {k: v for k, v in acc.items() if abs(v) > 1e-12}
    Lr, M, mono, col, val = L.symcon_plan_sym_table(plan, W)
    mine = {(int(Lr[i]), int(M[i]), tuple(int(x) for x in mono[i]), int(col[i])): val[i] for i in range(len(val))}
    assert set(mine) == set(acc)
    assert max(abs(mine[k] - acc[k]) for k in acc) < 1e-12
    L.symcon_destroy(plan)


def test_survey_counts(L):
    # symmetrised / folded nnz and monomials at lmax 3, corr 3
    expect = {(0,): (293, 94, 94), (0, 1): (1909, 410, 410), (0, 1, 2): (5911, 887, 743)}
    for outs, (nsym, nfold, nmono) in expect.items():
        plan = L.symcon_build_tables(3, 3, list(outs), 1, 1, -1)
        info = L.symcon_plan_info(plan)
        assert (info.n_sym_terms, info.n_fold, info.n_monomials) == (nsym, nfold, nmono)
        L.symcon_destroy(plan)


def test_generated_source_is_straight_line(L):
    plan = L.symcon_build_tables(3, 3, [0, 1], 1, 1, -1)
    src = L.symcon_plan_source(plan)
    for k in ("symcon_fold", "symcon_fwd", "symcon_bwd_dA", "symcon_bwd_dW", "symcon_unfold", "symcon_bwd2",
              "symcon_bwd2_dW"):
        assert f"void __launch_bounds__" in src and k in src
    assert src.count("fma2(") > 300
    L.symcon_destroy(plan)


def test_pack_matches_oracle(L):
    from oracle.packing import create_balanced_batches
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(0, 400))
        C = int(rng.integers(10, 300))
        G = int(rng.integers(1, 9))
        sizes = rng.integers(0, C + 1, size=n)
        offs, ids = L.symcon_pack_balanced(sizes, C, G)
        mine = [list(ids[offs[b]:offs[b + 1]]) for b in range(len(offs) - 1)]
        assert mine == create_balanced_batches([int(s) for s in sizes], C, G), trial
    with pytest.raises(L.SymconError):
        L.symcon_pack_balanced([3, 9], 8, 2)


def test_pack_table2_speed_and_balance(L):
    # ~1M graphs / ~100k batches in about one second on one CPU
    from synth.inputs import table2_sizes
    sizes = table2_sizes()
    t0 = time.time()
    offs, ids = L.symcon_pack_balanced(sizes, 3072, 8)
    dt = time.time() - t0
    loads = np.add.reduceat(sizes[ids], offs[:-1])
    assert len(offs) - 1 == 195144 and (len(offs) - 1) % 8 == 0
    assert loads.max() <= 3072 and np.sort(ids).tolist() == list(range(len(sizes)))
    assert dt < 2.65 * 1.5, dt     # 2.65M graphs: <= 1.5x the paper's per-graph rate


@pytest.mark.parametrize("lmax_y,hidden,lmax_out", [(3, (0, 1), 3), (3, (0,), 3), (2, (0, 1, 2), 2), (1, (1,), 1),
                                                    (3, (0, 1, 2, 3), 3)])
def test_tp_plan_paths_match_oracle(L, lmax_y, hidden, lmax_out):
    from oracle.tp import TPProblem
    prob = TPProblem(lmax_y, hidden, lmax_out)
    plan = L.symcon_tp_build(lmax_y, list(hidden), lmax_out, 8, -1)
    n_paths, n_y, n_h, n_out = L.symcon_tp_info(plan)
    assert (n_paths, n_y, n_h, n_out) == (prob.n_paths, prob.n_y, prob.n_h, prob.n_out)
    assert [L.symcon_tp_path(plan, p) for p in range(n_paths)] == [prob.path_l(p) for p in range(n_paths)]
    src = L.symcon_tp_source(plan)
    assert "symcon_tp_fwd" in src and "symcon_tp_bwd" in src
    with pytest.raises(L.SymconError):   # host-only plan cannot compute
        L.symcon_tp_forward(plan, 4, 4, 16, 16, 16, 16, 16, 16, 16, 1 << 20, None)
    L.symcon_tp_destroy(plan)


def test_tp_invalid_arguments(L):
    for args in [(4, [0], 3), (3, [1, 0], 3), (3, [], 3), (3, [0], 4), (0, [1], 0)]:
        with pytest.raises(L.SymconError) as e:
            L.symcon_tp_build(args[0], args[1], args[2], 8, -1)
        assert e.value.status == L.SYMCON_EINVAL


def test_peer_allreduce_argument_validation(L):
    # no device work: invalid arguments are rejected before any launch
    for bufs, rank in (([16] * 9, 0), ([16, 16], 2), ([16, 16], -1), ([], 0)):
        with pytest.raises(L.SymconError) as e:
            L.symcon_peer_allreduce(bufs, [16] * len(bufs), rank, 16, 1, 16, None, None)
        assert e.value.status == L.SYMCON_EINVAL
    with pytest.raises(L.SymconError):   # NULL peer pointer
        L.symcon_peer_allreduce([16, None], [16, 16], 0, 16, 1, 16, None, None)

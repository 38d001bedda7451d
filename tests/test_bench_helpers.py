"""bench.py's work accounting (CPU): the per-(node, channel) op counts and HBM bytes the roofline
fields are computed from."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@pytest.fixture(scope="module")
def L():
    from paper_2504_10700_b200 import build_lib
    build_lib.build()
    from paper_2504_10700_b200 import _lib
    return _lib


def test_alg_ops_matches_design_counts(L):
    import bench

    class S:
        pass
    sc = S()
    sc.plan = L.symcon_build_tables(3, 3, [0, 1], 89, 128, -1)
    ops = bench.alg_ops(sc)
    # DESIGN.md §7 table (MP-medium): Horner forward 705, reverse-Horner dW 731
    assert (ops["fwd"], ops["dA"], ops["dW"], ops["path"], ops["bwd2"], ops["bwd2_dW"]) == (705, 1486, 731, 2922, 3431, 1482)
    assert (ops["fwd_monomial_first"], ops["dW_monomial_first"], ops["path_monomial_first"]) == (888, 888, 3146)
    assert ops["n_fold"] == 410 and ops["prefixes"] == 123 and ops["deg3_monomials"] == 355
    L.symcon_destroy(sc.plan)


def test_tp_bytes_and_path_roofline():
    import bench
    from synth.inputs import CONFIGS
    f, b = bench.tp_bytes(50_000, 1_500_000, 128, 10, 4, 16, 16)
    # R (E K P floats) dominates: 7.68 GB read in the forward, read + written (dR) in the backward
    assert f == 4 * (1_500_000 * 128 * 10 + 50_000 * 128 * 4 + 1_500_000 * 16 + 50_000 * 128 * 16) + 8 * 1_500_000
    assert b - f == 4 * (1_500_000 * 16 + 50_000 * 128 * 4 + 1_500_000 * 128 * 10)

    class S:
        out_dim = 128 * 4
    r = bench.path_roofline(CONFIGS["mp_medium"], S(), 50_000, 3146 * 50_000 * 128, 1.2, False)
    assert r["bytes_per_node_channel"] == 224 and r["bound"] == "alu"
    assert abs(r["t_alu_ms"] - 3146 * 50_000 * 128 / (148 * 128 * 1.965e9) * 1e3) < 1e-9


def test_alg_ops_trie_generalises_alg_ops(L):
    """The prefix-trie counts (any degree; the correlation-4 bench lines) equal the degree-3 formulas
    exactly at correlation 3, and at correlation 4 the forward count is the trie size."""
    import bench

    class _P:
        pass
    for corr, outs in [(3, (0,)), (3, (0, 1)), (3, (0, 1, 2)), (4, (0,))]:
        s = _P()
        s.plan, s.correlation = L.symcon_build_tables(3, corr, list(outs), 1, 1, -1), corr
        t = bench.alg_ops_trie(s)
        if corr == 3:
            o = bench.alg_ops(s)
            assert all(t[k] == o[k] for k in ("fwd", "dA", "dW", "path")), (outs, t, o)
        else:
            assert t["fwd"] == t["trie_nodes"] and t["path"] == t["fwd"] + t["dA"] + t["dW"]
        L.symcon_destroy(s.plan)


def test_l2_flush_policy():
    """bench.py's L2 rule (the contract: flush L2 between timed steps or use inputs larger than L2):
    MP-medium 50k bins (512 MB of inputs per step) and OFF-small (131 MB > 126 MB) need no flush; the
    C = 3,072 pool (31 MB per step, 252 MB over 4 bins) is flushed."""
    import bench
    MB = 1e6
    assert not bench.needs_l2_flush(512 * MB, 4 * 1100 * MB)     # MP-medium, C = 50,000
    assert not bench.needs_l2_flush(131 * MB, 4 * 262 * MB)      # OFF-small molecule batches
    assert bench.needs_l2_flush(31 * MB, 252 * MB)               # C = 3,072
    assert not bench.needs_l2_flush(31 * MB, 400 * MB)           # a pool > 3x L2 evicts itself

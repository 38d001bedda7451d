"""Partition-quality study tooling (tools/partition_study.py): the
baseline packers and the metrics, on small instances with known answers."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import partition_study as ps  # noqa: E402


def _valid(bins, sizes, C, check_cap=True):
    ids = np.sort(np.concatenate(bins))
    assert (ids == np.arange(len(sizes))).all()          # Eq. (5): every graph exactly once
    if check_cap:
        assert all(sizes[b].sum() <= C for b in bins)     # Eq. (4)


def test_ffd_bfd_textbook_instance():
    # FFD on (7,5,5,4,3,2,2) with C=10 -> [7,3],[5,5],[4,2,2]: 3 bins (optimal); BFD the same
    sizes = np.array([5, 7, 2, 4, 3, 5, 2])
    for fn in (ps.pack_ffd, ps.pack_bfd):
        bins = fn(sizes, 10)
        _valid(bins, sizes, 10)
        assert len(bins) == 3
        assert sorted(sorted(sizes[b].tolist()) for b in bins) == [[2, 2, 4], [3, 7], [5, 5]]


def test_bfd_prefers_the_tightest_bin():
    sizes = np.array([6, 5, 4])        # after 6 and 5 (two bins, rem 4 and 5), BFD puts 4 into rem-4
    bins = ps.pack_bfd(sizes, 10)
    assert sorted(sorted(sizes[b].tolist()) for b in bins) == [[4, 6], [5]]
    bins = ps.pack_ffd(sizes, 10)      # FFD: first bin that fits -> also the 6-bin
    assert sorted(sorted(sizes[b].tolist()) for b in bins) == [[4, 6], [5]]


def test_fixed_count_and_metrics():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 100, 1000)
    bins = ps.pack_fixed_count(sizes, 500)
    _valid(bins, sizes, 500, check_cap=False)
    assert len({len(b) for b in bins[:-1]}) == 1           # a fixed number of graphs per batch
    m = ps.metrics(bins, sizes, ps.edges_of(sizes), 500, 4)
    assert m["bins_eq1"] == len(bins)
    # Eq. (2) as printed sums |V_i|^2 over all graphs: independent of the assignment
    assert np.isclose(m["padding_eq2"], (sizes.astype(float) ** 2).sum() / 500.0 ** 2)
    sq = [float((sizes[b].astype(float) ** 2).sum()) for b in bins]
    assert m["max_gap_eq3"] == max(sq) - min(sq)
    assert 0 < m["dp_efficiency_nodes"] <= 1


def test_alg1_balances_steps_better_than_ffd():
    from synth.inputs import table2_sizes
    sizes = table2_sizes(seed=0, scale=0.01)
    C, G = 50_000, 8
    e = ps.edges_of(sizes)
    a = ps.metrics(ps.pack_alg1(sizes, C, G), sizes, e, C, G)
    f = ps.metrics(ps.pack_ffd(sizes, C), sizes, e, C, G)
    assert a["over_capacity_bins"] == 0 and a["bins_eq1"] % G == 0
    assert a["max_gap_eq3"] < f["max_gap_eq3"]
    assert a["dp_efficiency_nodes"] >= f["dp_efficiency_nodes"]

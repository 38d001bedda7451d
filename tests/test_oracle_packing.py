"""Pins for oracle/packing.py (Alg. 1): hand trace, Eq. (4)/(5) properties, determinism."""
import json
import os

import numpy as np
import pytest

from oracle.packing import (create_balanced_batches, rank_schedule, eq1_num_bins, eq2_padding,
                            eq3_max_gap, eq4_capacity_ok, eq5_assignment_ok)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_trace():
    g = json.load(open(os.path.join(GOLD, "alg1_hand_trace.json")))
    bins = create_balanced_batches(g["sizes"], g["capacity"], g["gpus"])
    assert bins == g["bins"]
    assert [sum(g["sizes"][i] for i in b) for b in bins] == g["loads"]


@pytest.mark.parametrize("seed", range(30))
def test_properties_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    C = int(rng.integers(20, 200))
    G = int(rng.integers(1, 9))
    sizes = [int(x) for x in rng.integers(1, C + 1, size=n)]
    bins = create_balanced_batches(sizes, C, G)
    assert eq4_capacity_ok(bins, sizes, C)          # Eq. (4)
    assert eq5_assignment_ok(bins, n)               # Eq. (5)
    assert len(bins) % G == 0                       # M multiple of G (each recursion)
    assert eq1_num_bins(bins) >= -(-sum(sizes) // C)
    assert bins == create_balanced_batches(sizes, C, G)   # deterministic (stable sorts)
    assert eq2_padding(bins, sizes, C) == pytest.approx(sum(s * s for s in sizes) / C ** 2)
    assert eq3_max_gap(bins, sizes) >= 0


def test_eq2_eq3_hand_trace_values():
    """Eq. (2) and Eq. (3) on the hand-traced Alg. 1 plan of
    tests/golden/alg1_hand_trace.json, worked by hand (W = C = 8):
      Eq. (2) = (7^2 + 5^2 + 4^2 + 3^2 + 2^2 + 1^2) / 8^2 = 104 / 64 = 1.625
      Eq. (3): squared loads per bin {7}->49, {5}->25, {4,1}->17, {3,2}->13; max gap 49 - 13 = 36.
    A dropped square (Eq. 2 -> 22/64, Eq. 3 -> 7 - 5 = 2), a missing /W^2 or a max-only Eq. (3)
    fails here."""
    g = json.load(open(os.path.join(GOLD, "alg1_hand_trace.json")))
    bins = create_balanced_batches(g["sizes"], g["capacity"], g["gpus"])
    assert eq2_padding(bins, g["sizes"], g["capacity"]) == 1.625
    assert eq3_max_gap(bins, g["sizes"]) == 36
    # a worse plan of the same graphs has a larger Eq. (3) gap: {7,1} {5,3} {4,2} {} -> 50, 34, 20, 0
    assert eq3_max_gap([[0, 5], [1, 3], [2, 4], []], g["sizes"]) == 50
    assert eq1_num_bins([[0, 5], [1, 3], [2, 4], []]) == 3


def test_oversize_rejected_and_empty():
    with pytest.raises(ValueError):
        create_balanced_batches([5, 9], 8, 2)
    assert create_balanced_batches([], 8, 2) == []


def test_rank_schedule_round_robin():
    assert rank_schedule(6, 2) == [(0, 0), (1, 0), (0, 1), (1, 1), (0, 2), (1, 2)]


def test_table2_sample_balance():
    from synth.inputs import table2_sizes
    sizes = [int(x) for x in table2_sizes(scale=0.01)]
    C = 3072
    bins = create_balanced_batches(sizes, C, 4)
    loads = np.array([sum(sizes[i] for i in b) for b in bins])
    assert loads.max() <= C and eq5_assignment_ok(bins, len(sizes))
    # every non-final bin ends within the largest graph of full
    assert np.sort(loads)[len(loads) // 10] >= C - 768

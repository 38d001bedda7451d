"""Alg. 1 Create-Balanced-Batches and the Eq. (1)-(5) metrics (oracle; tests only).

Follows PAPER.md:365-411 line by line with DESIGN.md's readings:
  s14 final version (with second chance), not the draft;
  s15 second chance fires when min remaining(non-full) < max remaining(full),
      the full set is cumulative across rounds, and all full bins are unmarked;
  s16 graphs sorted by size descending then index ascending; bins by remaining
      capacity descending then creation order;
  s17 a graph larger than C is rejected (ValueError);
  s18 bin j runs on rank j mod G at step j // G.
"""
from math import ceil


class _Bin:
    __slots__ = ("id", "cap", "items", "full")

    def __init__(self, bid, cap):
        self.id, self.cap, self.items, self.full = bid, cap, [], False


def create_balanced_batches(sizes, C, G, _ids=None, _next_id=0):
    """Returns a list of bins (lists of original graph indices) in creation order."""
    if _ids is None:
        if any(s > C for s in sizes):
            raise ValueError("graph larger than bin capacity")  # reading s17
        if any(s < 0 for s in sizes):
            raise ValueError("negative size")
        order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))   # line 1, StableSort
        Ls = [sizes[i] for i in order]
        I = order
    else:
        Ls, I = list(sizes), list(_ids)
    N = len(Ls)
    if N == 0:
        return []
    S = sum(Ls)                                                           # line 2
    M = ceil(S / C)                                                       # line 3
    M = ceil(M / G) * G                                                   # line 4
    M = max(M, G)
    bins = [_Bin(_next_id + j, C) for j in range(M)]                      # line 5
    active = list(bins)
    full_set = []
    p = 0                                                                 # line 6
    while p < N and active:                                               # line 7
        active.sort(key=lambda b: (-b.cap, b.id))                         # line 8
        for b in active:                                                  # line 9
            if b.cap >= Ls[p]:                                            # line 10
                b.items.append(I[p])                                      # line 11
                b.cap -= Ls[p]                                            # line 12
                p += 1                                                    # line 13
                if p >= N:                                                # line 14
                    break
            else:
                b.full = True                                             # line 17
        newly_full = [b for b in active if b.full]                        # line 18
        active = [b for b in active if not b.full]                        # line 19
        full_set.extend(newly_full)
        if active and full_set and min(b.cap for b in active) < max(b.cap for b in full_set):  # line 20
            for b in full_set:                                            # line 21
                b.full = False
            active = active + full_set                                    # line 22
            full_set = []
    out = [b.items for b in bins]
    if p < N:                                                             # line 23
        out += create_balanced_batches(Ls[p:], C, G, _ids=I[p:], _next_id=_next_id + M)  # line 24-25
    return out


def rank_schedule(n_bins, G):
    """Reading s18: bin j -> (rank j % G, step j // G)."""
    return [(j % G, j // G) for j in range(n_bins)]


# ---------------------------------------------------------------- Eq. (1)-(5)
def eq1_num_bins(bins):
    """Eq. (1): number of used bins."""
    return sum(1 for b in bins if b)


def eq2_padding(bins, sizes, C):
    """Eq. (2): sum_j sum_i b_ij |V_i|^2 / W^2 with W = C."""
    return sum(sizes[i] ** 2 for b in bins for i in b) / float(C * C)


def eq3_max_gap(bins, sizes):
    """Eq. (3): max_{j,k} |sum_i b_ij |V_i|^2 - sum_i b_ik |V_i|^2|."""
    loads = [sum(sizes[i] ** 2 for i in b) for b in bins]
    return max(loads) - min(loads) if loads else 0


def eq4_capacity_ok(bins, sizes, C):
    """Eq. (4): sum_i |V_i| b_ij <= C a_j."""
    return all(sum(sizes[i] for i in b) <= C for b in bins)


def eq5_assignment_ok(bins, n):
    """Eq. (5): every graph in exactly one bin."""
    seen = [0] * n
    for b in bins:
        for i in b:
            seen[i] += 1
    return all(s == 1 for s in seen)

// Alg. 1 Create-Balanced-Batches, host C++ (SURVEY.md §8(a) step a7).
// Readings: s14 final version with second chance; s15 cumulative full set,
// trigger min remaining(non-full) < max remaining(full), unmark all; s16 graphs by
// (size desc, index asc), bins by (remaining desc, creation order); s17 oversize rejected by
// the caller; the recursion on leftovers (lines 23-25) is the outer loop below.
// Complexity O(N log N) + O(rounds * M log M).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "internal.h"

namespace symcon {

int64_t pack_balanced(const int64_t* sizes, int64_t n, int64_t C, int G, std::vector<std::vector<int64_t>>& bins) {
  bins.clear();
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sizes[a] > sizes[b]; });  // line 1
  int64_t p = 0;
  while (p < n) {
    int64_t S = 0;
    for (int64_t q = p; q < n; q++) S += sizes[order[q]];                 // line 2 (remaining items)
    int64_t M = (S + C - 1) / C;                                          // line 3
    M = (M + G - 1) / G * G;                                              // line 4
    if (M < G) M = G;
    const int64_t first = (int64_t)bins.size();
    bins.resize(first + M);                                               // line 5
    std::vector<int64_t> cap(M, C);
    std::vector<int64_t> active(M);
    std::iota(active.begin(), active.end(), 0);
    std::vector<char> full(M, 0);
    std::vector<int64_t> full_set;
    int64_t full_max = -1;
    auto by_cap = [&](int64_t a, int64_t b) { return cap[a] != cap[b] ? cap[a] > cap[b] : a < b; };
    while (p < n && !active.empty()) {                                    // line 7
      std::sort(active.begin(), active.end(), by_cap);                    // line 8 (keyed, so stable)
      for (int64_t b : active) {                                          // line 9
        const int64_t l = sizes[order[p]];
        if (cap[b] >= l) {                                                // line 10
          bins[first + b].push_back(order[p]);                            // line 11
          cap[b] -= l;                                                    // line 12
          if (++p >= n) break;                                            // lines 13-15
        } else {
          full[b] = 1;                                                    // line 17
        }
      }
      std::vector<int64_t> still;                                         // lines 18-19
      still.reserve(active.size());
      for (int64_t b : active) {
        if (full[b]) { full_set.push_back(b); full_max = std::max(full_max, cap[b]); }
        else still.push_back(b);
      }
      active.swap(still);
      if (!active.empty() && !full_set.empty()) {                          // line 20
        int64_t mn = cap[active[0]];
        for (int64_t b : active) mn = std::min(mn, cap[b]);
        if (mn < full_max) {                                              // lines 21-22
          for (int64_t b : full_set) { full[b] = 0; active.push_back(b); }
          full_set.clear();
          full_max = -1;
        }
      }
    }
  }                                                                       // lines 23-25: recurse on the rest
  return (int64_t)bins.size();
}

}  // namespace symcon

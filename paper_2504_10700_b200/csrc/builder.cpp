// Host U-table builder ("sparsity pattern is
// deterministic and known at compile time", "pre-compute all valid
// combinations, store only non-zero coefficients, and create lookup tables").
//
// 1. Paths: for each output L and nu = 1..corr, left-nested coupling trees
//    (l1 (x) l2 -> L2, L2 (x) l3 -> L3, ...), every intermediate allowed, last = L, kept iff
//    sum(l) + L is even (DESIGN.md §3 readings s4, s9); eta order = lexicographic on the
//    interleaved key (l1, l2, L2, l3, L3) — the nested loops below generate exactly that order.
// 2. U_{nu,L,eta}[M, t1..t_nu] = chain of pairwise real couplings (cg.cpp).
// 3. Symmetrise to sorted monomials: U~[(L,M,mono), path] = sum over ordered tuples t that
//    sort to mono of U[M,t]. B only sees U~ because prod_j A[t_j] depends on the multiset.
// 4. Rows (L,M,mono) are put in codegen order: degree-1 rows, then per prefix (a,b):
//    the degree-2 row(s) (a,b) followed by degree-3 rows (a,b,c), c ascending, each followed by
//    its degree-4 rows (a,b,c,d), d ascending (correlation 4).
#include <algorithm>
#include <cmath>
#include <map>

#include "internal.h"

namespace symcon {
namespace {

void enumerate(int lmax, int nu, int L, std::vector<PathDesc>& out) {
  auto keep = [&](int s) { return (s + L) % 2 == 0; };
  if (nu == 1) {
    if (L <= lmax) {
      PathDesc p;
      p.L = L; p.nu = 1; p.ls[0] = L;
      out.push_back(p);
    }
    return;
  }
  // nu = 4 (correlation 4, reading s4b): every intermediate L_j has natural parity,
  // (L_j + l_1 + ... + l_j) even, and L_j <= 11 (the coupling tables stop at 3 + 3 + 3 + 3 - 1)
  auto nat = [&](int Lj, int s) { return nu < 4 || ((Lj + s) % 2 == 0 && Lj < 12); };
  for (int l1 = 0; l1 <= lmax; l1++)
    for (int l2 = 0; l2 <= lmax; l2++)
      for (int L2 = std::abs(l1 - l2); L2 <= l1 + l2; L2++) {
        if (nu == 2) {
          if (L2 == L && keep(l1 + l2)) {
            PathDesc p;
            p.L = L; p.nu = 2; p.ls = {l1, l2, -1, -1}; p.mids = {L2, -1, -1};
            out.push_back(p);
          }
          continue;
        }
        if (!nat(L2, l1 + l2)) continue;
        for (int l3 = 0; l3 <= lmax; l3++)
          for (int L3 = std::abs(L2 - l3); L3 <= L2 + l3; L3++) {
            if (nu == 3) {
              if (L3 == L && keep(l1 + l2 + l3)) {
                PathDesc p;
                p.L = L; p.nu = 3; p.ls = {l1, l2, l3, -1}; p.mids = {L2, L3, -1};
                out.push_back(p);
              }
              continue;
            }
            if (!nat(L3, l1 + l2 + l3)) continue;
            for (int l4 = 0; l4 <= lmax; l4++)
              for (int L4 = std::abs(L3 - l4); L4 <= L3 + l4; L4++)
                if (L4 == L && keep(l1 + l2 + l3 + l4)) {
                  PathDesc p;
                  p.L = L; p.nu = 4; p.ls = {l1, l2, l3, l4}; p.mids = {L2, L3, L4};
                  out.push_back(p);
                }
          }
      }
}

inline int lmi(int l, int m) { return l * l + l + m; }

}  // namespace

bool build_tables(int lmax_in, int corr, const std::vector<int>& out_L, int E, int K, Tables& t) {
  t.lmax_in = lmax_in;
  t.corr = corr;
  t.n_lm = (lmax_in + 1) * (lmax_in + 1);
  t.E = E;
  t.K = K;
  t.out_L = out_L;
  t.out_off.clear();
  int off = 0;
  for (int L : out_L) { t.out_off.push_back(off); off += 2 * L + 1; }
  t.out_per_ch = off;
  t.paths.clear();
  for (int L : out_L)
    for (int nu = 1; nu <= corr; nu++) {
      std::vector<PathDesc> ps;
      enumerate(lmax_in, nu, L, ps);
      for (size_t e = 0; e < ps.size(); e++) {
        ps[e].eta = (int)e;
        ps[e].col = (int)t.paths.size();
        t.paths.push_back(ps[e]);
      }
    }
  // symmetrised accumulation: key (out index, M, mono) -> col -> value
  std::map<std::tuple<int, int, std::array<int, 4>>, std::map<int, double>> acc;
  t.n_raw_terms = 0;
  for (const auto& p : t.paths) {
    int oi = (int)(std::find(out_L.begin(), out_L.end(), p.L) - out_L.begin());
    const int nL = 2 * p.L + 1;
    // T[Mj][m1..mj] dense, built left to right
    int cur = p.ls[0];
    std::vector<double> T((2 * cur + 1) * (2 * cur + 1), 0.0);
    for (int i = 0; i < 2 * cur + 1; i++) T[i * (2 * cur + 1) + i] = 1.0;
    int inner = 2 * cur + 1;  // product of (2 l_j + 1) so far
    for (int j = 1; j < p.nu; j++) {
      int lj = p.ls[j], Lj = p.mids[j - 1];
      auto C = real_coupling(cur, lj, Lj);  // [Lj][cur][lj]
      const int nLj = 2 * Lj + 1, nc = 2 * cur + 1, nl = 2 * lj + 1;
      std::vector<double> T2(nLj * inner * nl, 0.0);
      for (int Mj = 0; Mj < nLj; Mj++)
        for (int Mc = 0; Mc < nc; Mc++)
          for (int ml = 0; ml < nl; ml++) {
            double c = C[(Mj * nc + Mc) * nl + ml];
            if (c == 0.0) continue;
            for (int r = 0; r < inner; r++) {
              double x = T[Mc * inner + r];
              if (x != 0.0) T2[(Mj * inner + r) * nl + ml] += c * x;
            }
          }
      T.swap(T2);
      inner *= nl;
      cur = Lj;
    }
    if (cur != p.L) { set_error("internal: path does not end in L"); return false; }
    // walk nonzeros
    for (int M = 0; M < nL; M++)
      for (int r = 0; r < inner; r++) {
        double u = T[M * inner + r];
        if (std::abs(u) <= 1e-13) continue;
        t.n_raw_terms++;
        std::array<int, 4> tup{{-1, -1, -1, -1}};
        int rem = r;
        for (int j = p.nu - 1; j >= 0; j--) {
          int nl = 2 * p.ls[j] + 1;
          int mj = rem % nl;
          rem /= nl;
          tup[j] = lmi(p.ls[j], mj - p.ls[j]);
        }
        std::sort(tup.begin(), tup.begin() + p.nu);
        acc[{oi, M - p.L, tup}][p.col] += u;
      }
  }
  // collect rows, drop vanishing entries
  struct Tmp { SymRow row; };
  std::vector<SymRow> rows;
  t.n_sym_terms = 0;
  for (auto& kv : acc) {
    SymRow s;
    int oi = std::get<0>(kv.first);
    s.L = out_L[oi];
    s.M = std::get<1>(kv.first);
    s.out = t.out_off[oi] + s.M + s.L;
    s.mono = std::get<2>(kv.first);
    s.deg = (s.mono[0] >= 0) + (s.mono[1] >= 0) + (s.mono[2] >= 0) + (s.mono[3] >= 0);
    for (auto& cv : kv.second)
      if (std::abs(cv.second) > 1e-12) s.cols.push_back({cv.first, cv.second});
    if (s.cols.empty()) continue;
    t.n_sym_terms += (int64_t)s.cols.size();
    rows.push_back(s);
  }
  // codegen order
  auto key = [](const SymRow& s) {
    // deg-1 first (group -1), then prefix (a,b) groups, inside: deg2 before deg3 (c asc), each
    // deg-3 row (a,b,c) before its deg-4 extensions (a,b,c,d), d asc (monomials padded with -1)
    int a = s.mono[0], b = s.deg >= 2 ? s.mono[1] : -1;
    int grp = (s.deg == 1) ? -1 : a * 64 + b;
    return std::make_tuple(grp, s.deg == 1 ? a : s.mono[2], s.mono[3], s.out);
  };
  std::stable_sort(rows.begin(), rows.end(), [&](const SymRow& x, const SymRow& y) { return key(x) < key(y); });
  t.rows = rows;
  std::map<std::array<int, 4>, int> monos;
  for (auto& r : t.rows) monos[r.mono] = 1;
  t.n_monomials = (int)monos.size();
  return true;
}

}  // namespace symcon

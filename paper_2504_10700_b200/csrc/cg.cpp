// Pairwise real Clebsch-Gordan coupling for the U-table builder (product side).
//
// Construction (independent of the oracle's Racah sum): complex CG by the ladder-operator
// method — for each J from j1+j2 down, the top state |J J> is the unit vector in the M=J
// subspace orthogonal to every |J' J>, J' > J (Condon-Shortley: <j1 j1; j2 J-j1|J J> > 0),
// lowered with J- = J1- + J2-. Selection rules of PAPER.md:696-697 hold by construction
// (only m1+m2=M product states are ever touched, J runs over the triangle range).
// Then the DESIGN.md §3 real basis change, global-phase removal, and the sign rule
// "first entry with |x| > 1e-12 in row-major [M][m1][m2] order is positive".
#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"

namespace symcon {
namespace {

// complex CG table for (j1, j2): cg[J][M+J][m1+j1] (m2 = M - m1)
struct ComplexCG {
  int j1, j2;
  std::vector<std::vector<std::vector<double>>> c;  // [J][M+J][m1+j1]
};

ComplexCG ladder_cg(int j1, int j2) {
  ComplexCG r;
  r.j1 = j1;
  r.j2 = j2;
  const int Jmax = j1 + j2, Jmin = std::abs(j1 - j2);
  r.c.assign(Jmax + 1, {});
  // state vector over m1 in [-j1, j1] for fixed M (entries with |M-m1| > j2 are zero)
  for (int J = Jmax; J >= Jmin; --J) {
    std::vector<std::vector<double>> st(2 * J + 1, std::vector<double>(2 * j1 + 1, 0.0));
    // top state M = J
    std::vector<double> v(2 * j1 + 1, 0.0);
    v[j1 + j1] = (std::abs(J - j1) <= j2) ? 1.0 : 0.0;
    for (int Jp = Jmax; Jp > J; --Jp) {  // project out |Jp, J>
      const auto& u = r.c[Jp][J + Jp];
      double d = 0;
      for (int i = 0; i < 2 * j1 + 1; i++) d += u[i] * v[i];
      for (int i = 0; i < 2 * j1 + 1; i++) v[i] -= d * u[i];
    }
    double nrm = 0;
    for (double x : v) nrm += x * x;
    nrm = std::sqrt(nrm);
    for (double& x : v) x /= nrm;
    st[2 * J] = v;
    // lower: |J, M-1> = J- |J, M> / sqrt((J+M)(J-M+1))
    for (int M = J; M > -J; --M) {
      std::vector<double> w(2 * j1 + 1, 0.0);
      const auto& cur = st[M + J];
      for (int m1 = -j1; m1 <= j1; m1++) {
        int m2 = M - m1;
        double a = cur[m1 + j1];
        if (a == 0.0 || std::abs(m2) > j2) continue;
        if (m1 - 1 >= -j1) w[m1 - 1 + j1] += a * std::sqrt(double((j1 + m1) * (j1 - m1 + 1)));
        if (m2 - 1 >= -j2) w[m1 + j1] += a * std::sqrt(double((j2 + m2) * (j2 - m2 + 1)));
      }
      double s = std::sqrt(double((J + M) * (J - M + 1)));
      for (double& x : w) x /= s;
      st[M - 1 + J] = w;
    }
    r.c[J] = st;
  }
  return r;
}

// Q_l: Y_real = Q_l Y_complex  (rows real m, cols complex m), DESIGN.md §3
std::vector<std::complex<double>> real_from_complex(int l) {
  const int n = 2 * l + 1;
  std::vector<std::complex<double>> Q(n * n, 0.0);
  const double r = 1.0 / std::sqrt(2.0);
  const std::complex<double> I(0.0, 1.0);
  for (int m = -l; m <= l; m++) {
    int row = m + l;
    double sgn = (m % 2 == 0) ? 1.0 : -1.0;  // (-1)^m
    if (m < 0) {
      Q[row * n + (m + l)] += I * r;
      Q[row * n + (-m + l)] += -I * r * sgn;
    } else if (m == 0) {
      Q[row * n + l] = 1.0;
    } else {
      Q[row * n + (-m + l)] += r;
      Q[row * n + (m + l)] += r * sgn;
    }
  }
  return Q;
}

std::mutex g_mu;
std::map<std::tuple<int, int, int>, std::vector<double>> g_cache;

}  // namespace

std::vector<double> real_coupling(int l1, int l2, int L) {
  const int nL = 2 * L + 1, n1 = 2 * l1 + 1, n2 = 2 * l2 + 1;
  std::vector<double> out(nL * n1 * n2, 0.0);
  if (L < std::abs(l1 - l2) || L > l1 + l2) return out;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_cache.find({l1, l2, L});
    if (it != g_cache.end()) return it->second;
  }
  ComplexCG cg = ladder_cg(l1, l2);
  auto QL = real_from_complex(L), Q1 = real_from_complex(l1), Q2 = real_from_complex(l2);
  // C_real[M,a,b] = sum QL[M,M'] CG[M',m1',m2'] conj(Q1[a,m1']) conj(Q2[b,m2'])
  std::vector<std::complex<double>> cr(nL * n1 * n2, 0.0);
  for (int Mp = -L; Mp <= L; Mp++)
    for (int m1 = -l1; m1 <= l1; m1++) {
      int m2 = Mp - m1;
      if (std::abs(m2) > l2) continue;
      double c = cg.c[L][Mp + L][m1 + l1];
      if (c == 0.0) continue;
      for (int M = 0; M < nL; M++) {
        auto qM = QL[M * nL + (Mp + L)];
        if (qM == 0.0) continue;
        for (int a = 0; a < n1; a++) {
          auto qa = std::conj(Q1[a * n1 + (m1 + l1)]);
          if (qa == 0.0) continue;
          for (int b = 0; b < n2; b++) {
            auto qb = std::conj(Q2[b * n2 + (m2 + l2)]);
            if (qb == 0.0) continue;
            cr[(M * n1 + a) * n2 + b] += qM * c * qa * qb;
          }
        }
      }
    }
  // global phase: the coupling is either purely real or purely imaginary
  double re = 0, im = 0;
  for (auto& z : cr) { re += z.real() * z.real(); im += z.imag() * z.imag(); }
  for (size_t i = 0; i < cr.size(); i++) out[i] = (re >= im) ? cr[i].real() : cr[i].imag();
  for (double& x : out)
    if (std::abs(x) < 1e-12) x = 0.0;
  for (double x : out)
    if (x != 0.0) {
      if (x < 0)
        for (double& y : out) y = -y;
      break;
    }
  std::lock_guard<std::mutex> g(g_mu);
  g_cache[{l1, l2, L}] = out;
  return out;
}

}  // namespace symcon

/* ORACLE C evaluator — test infrastructure only (see oracle/__init__.py).
 *
 * A plain fp64 loop over the raw ordered-tuple nonzeros that oracle/paths.py
 * builds (this file builds no tables of its own and shares nothing with the
 * CUDA product). It evaluates exactly the definitions in oracle/contraction.py
 * (Alg. 3; Eq. (2); forces as derivatives,
 * PAPER.md:331), parallel over nodes with OpenMP, so that the oracle can be
 * timed on the host cores and checked at full BASELINE sizes.
 *
 * Term table (one row per raw nonzero U entry, built by oracle/ceval.py):
 *   col[t]    W column (path)
 *   nu[t]     order 1..4                tup[4t..4t+3] lm indices (unused slots 0)
 *   u[t]      U value
 * Output addressing: B[i*out_dim + blk[t]*K + k*wid[t] + mpos[t]].
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int64_t n_terms, n_lm, out_per_ch, n_paths;
  const int32_t *col, *nu, *tup, *blk, *wid, *mpos;
  const double* u;
} oracle_tables;

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* B[N][out_dim] (overwritten). A [N][K][n_lm], W [E][P][K] as float32 inputs. */
void oracle_forward(const oracle_tables* T, int64_t N, int64_t K, const float* A, const float* W,
                    const int32_t* node_elem, double* B) {
  int64_t i;
#pragma omp parallel for schedule(dynamic, 16)
  for (i = 0; i < N; i++) {
    const int64_t z = node_elem[i];
    const int64_t out_dim = T->out_per_ch * K;
    double* Bi = B + i * out_dim;
    memset(Bi, 0, sizeof(double) * out_dim);
    for (int64_t k = 0; k < K; k++) {
      const float* a = A + (i * K + k) * T->n_lm;
      for (int64_t t = 0; t < T->n_terms; t++) {
        double prod = T->u[t];
        for (int j = 0; j < T->nu[t]; j++) prod *= (double)a[T->tup[4 * t + j]];
        double w = (double)W[(z * T->n_paths + T->col[t]) * K + k];
        Bi[T->blk[t] * K + k * T->wid[t] + T->mpos[t]] += w * prod;
      }
    }
  }
}

/* dA [N][K][n_lm] and dW [E][P][K] (both overwritten; either may be NULL). */
void oracle_backward(const oracle_tables* T, int64_t N, int64_t K, int64_t E, const float* A,
                     const float* W, const int32_t* node_elem, const float* dB, double* dA, double* dW) {
  const int64_t wsz = E * T->n_paths * K;
  int nth = oracle_num_threads();
  double* priv = NULL;
  if (dW) {
    priv = (double*)calloc((size_t)nth * (size_t)wsz, sizeof(double));
  }
#pragma omp parallel
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* myW = priv ? priv + (size_t)tid * wsz : NULL;
    int64_t i;
#pragma omp for schedule(dynamic, 16)
    for (i = 0; i < N; i++) {
      const int64_t z = node_elem[i];
      if (dA) memset(dA + i * K * T->n_lm, 0, sizeof(double) * K * T->n_lm);
      for (int64_t k = 0; k < K; k++) {
        const float* a = A + (i * K + k) * T->n_lm;
        double* da = dA ? dA + (i * K + k) * T->n_lm : NULL;
        for (int64_t t = 0; t < T->n_terms; t++) {
          double g = (double)dB[i * T->out_per_ch * K + T->blk[t] * K + k * T->wid[t] + T->mpos[t]];
          double w = (double)W[(z * T->n_paths + T->col[t]) * K + k];
          int nu = T->nu[t];
          const int32_t* tp = T->tup + 4 * t;
          if (myW) {
            double prod = T->u[t];
            for (int j = 0; j < nu; j++) prod *= (double)a[tp[j]];
            myW[(z * T->n_paths + T->col[t]) * K + k] += g * prod;
          }
          if (da) {
            for (int j = 0; j < nu; j++) {
              double part = g * w * T->u[t];
              for (int jj = 0; jj < nu; jj++)
                if (jj != j) part *= (double)a[tp[jj]];
              da[tp[j]] += part;
            }
          }
        }
      }
    }
  }
  if (dW) {
    memset(dW, 0, sizeof(double) * wsz);
    for (int t = 0; t < nth; t++)
      for (int64_t x = 0; x < wsz; x++) dW[x] += priv[(size_t)t * wsz + x];
    free(priv);
  }
}

/* Double backward (oracle/contraction.py:backward2): derivatives of <uA, dA(A, W, dB)> with
 * respect to dB (dB_bar [N][out_dim]), A (A_bar [N][K][n_lm]) and W (W_bar [E][P][K]); all
 * overwritten, any may be NULL. Per raw term t with product prod_j a[t_j]:
 *   jvp = sum_j uA[t_j] prod_{j' != j} a[t_j']
 *   dB_bar[out(t)] += w u jvp;  W_bar[z, col] += g u jvp
 *   A_bar[t_j2]    += g w u uA[t_j] prod_{j' not in {j, j2}} a[t_j']   (j != j2) */
void oracle_backward2(const oracle_tables* T, int64_t N, int64_t K, int64_t E, const float* A,
                      const float* W, const int32_t* node_elem, const float* dB, const float* uA,
                      double* dB_bar, double* A_bar, double* W_bar) {
  const int64_t wsz = E * T->n_paths * K;
  const int64_t out_dim = T->out_per_ch * K;
  int nth = oracle_num_threads();
  double* priv = NULL;
  if (W_bar) priv = (double*)calloc((size_t)nth * (size_t)wsz, sizeof(double));
#pragma omp parallel
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* myW = priv ? priv + (size_t)tid * wsz : NULL;
    int64_t i;
#pragma omp for schedule(dynamic, 16)
    for (i = 0; i < N; i++) {
      const int64_t z = node_elem[i];
      if (A_bar) memset(A_bar + i * K * T->n_lm, 0, sizeof(double) * K * T->n_lm);
      if (dB_bar) memset(dB_bar + i * out_dim, 0, sizeof(double) * out_dim);
      for (int64_t k = 0; k < K; k++) {
        const float* a = A + (i * K + k) * T->n_lm;
        const float* ua = uA + (i * K + k) * T->n_lm;
        double* ab = A_bar ? A_bar + (i * K + k) * T->n_lm : NULL;
        for (int64_t t = 0; t < T->n_terms; t++) {
          const int64_t o = i * out_dim + T->blk[t] * K + k * T->wid[t] + T->mpos[t];
          double g = (double)dB[o];
          double w = (double)W[(z * T->n_paths + T->col[t]) * K + k];
          int nu = T->nu[t];
          const int32_t* tp = T->tup + 4 * t;
          double jvp = 0.0;
          for (int j = 0; j < nu; j++) {
            double part = (double)ua[tp[j]];
            for (int jj = 0; jj < nu; jj++)
              if (jj != j) part *= (double)a[tp[jj]];
            jvp += part;
          }
          if (dB_bar) dB_bar[o] += w * T->u[t] * jvp;
          if (myW) myW[(z * T->n_paths + T->col[t]) * K + k] += g * T->u[t] * jvp;
          if (ab) {
            for (int j = 0; j < nu; j++)
              for (int j2 = 0; j2 < nu; j2++) {
                if (j2 == j) continue;
                double part = g * w * T->u[t] * (double)ua[tp[j]];
                for (int jj = 0; jj < nu; jj++)
                  if (jj != j && jj != j2) part *= (double)a[tp[jj]];
                ab[tp[j2]] += part;
              }
          }
        }
      }
    }
  }
  if (W_bar) {
    memset(W_bar, 0, sizeof(double) * wsz);
    for (int t = 0; t < nth; t++)
      for (int64_t x = 0; x < wsz; x++) W_bar[x] += priv[(size_t)t * wsz + x];
    free(priv);
  }
}

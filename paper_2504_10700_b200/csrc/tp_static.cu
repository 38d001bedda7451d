// Static (nvcc) kernels of the channelwise tensor product: receiver CSR
// with input validation, a deterministic sender CSR (counting sort + per-segment sort by edge id)
// and the fixed-order reduction of per-edge dh contributions onto the senders.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace symcon {
namespace {

__global__ void tp_check(const int* __restrict__ sender, const int* __restrict__ receiver, int N, int E,
                         unsigned long long* err) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int r = receiver[e], s = sender[e];
    const bool bad = r < 0 || r >= N || s < 0 || s >= N || (e > 0 && receiver[e - 1] > r);
    if (bad) atomicMin(err, (unsigned long long)e);
  }
}

// recv_off[i] = first edge with receiver >= i (lower bound), i in [0, N]
__global__ void tp_recv_off(const int* __restrict__ receiver, int N, int E, int* __restrict__ recv_off) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= N; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = E;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (receiver[mid] < i) lo = mid + 1; else hi = mid;
    }
    recv_off[i] = lo;
  }
}

__global__ void tp_send_hist(const int* __restrict__ sender, int N, int E, int* __restrict__ cnt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int s = sender[e];
    if (s >= 0 && s < N) atomicAdd(cnt + s, 1);
  }
}

// single-block exclusive scan of cnt[N] -> off[N+1] and cur[N] (= off[0..N))
__global__ void __launch_bounds__(1024) tp_scan(const int* __restrict__ cnt, int N, int* __restrict__ off,
                                                 int* __restrict__ cur) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < N; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < N ? cnt[i] : 0;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = warp_sums[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
    if (i < N) { off[i] = excl; cur[i] = excl; }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[N] = carry;
}

__global__ void tp_send_scatter(const int* __restrict__ sender, int N, int E, int* __restrict__ cur,
                                int* __restrict__ perm) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int s = sender[e];
    if (s >= 0 && s < N) perm[atomicAdd(cur + s, 1)] = e;
  }
}

// each sender's edge list sorted by edge id (deterministic order for the dh reduction)
__global__ void tp_seg_sort(const int* __restrict__ off, int N, int* __restrict__ perm) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    const int a = off[j], b = off[j + 1];
    for (int q = a + 1; q < b; q++) {
      const int v = perm[q];
      int t = q - 1;
      while (t >= a && perm[t] > v) { perm[t + 1] = perm[t]; t--; }
      perm[t + 1] = v;
    }
  }
}

// dh[j][:][k] = sum over the sender's edges (ascending id) of their dhe rows, which the backward
// kernel wrote at the edge's position in the sender CSR (contiguous per sender); thread per (j,
// channel pair) with 8-byte loads (K even) or per (j, channel); summation order fixed.
template <int CPT, int NH>
__global__ void tp_dh_reduce(const float* __restrict__ dhe, const int* __restrict__ off, int N, int K,
                             float* __restrict__ dh) {
  const int KT = K / CPT;
  const long long total = (long long)N * KT;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / KT), k = (int)(t - (long long)j * KT) * CPT;
    float acc[NH][CPT];
#pragma unroll
    for (int q = 0; q < NH; q++)
#pragma unroll
      for (int c = 0; c < CPT; c++) acc[q][c] = 0.f;
    const int a = off[j], b = off[j + 1];
    for (int s0 = a; s0 < b; s0 += 4) {
      float v[4][NH][CPT];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const bool ok = s0 + u < b;
        const float* src = dhe + (long long)(ok ? s0 + u : a) * NH * K + k;
#pragma unroll
        for (int q = 0; q < NH; q++) {
          if (CPT == 2) {
            const float2 x = ok ? __ldg(reinterpret_cast<const float2*>(src + (long long)q * K)) : make_float2(0.f, 0.f);
            v[u][q][0] = x.x;
            v[u][q][CPT - 1] = x.y;
          } else {
            v[u][q][0] = ok ? __ldg(src + (long long)q * K) : 0.f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int q = 0; q < NH; q++)
#pragma unroll
          for (int c = 0; c < CPT; c++) acc[q][c] += v[u][q][c];
    }
    float* d = dh + (long long)j * NH * K + k;   // dh[j][q][k] (h's layout)
#pragma unroll
    for (int q = 0; q < NH; q++) {
      if (CPT == 2) *reinterpret_cast<float2*>(d + (long long)q * K) = make_float2(acc[q][0], acc[q][CPT - 1]);
      else d[(long long)q * K] = acc[q][0];
    }
  }
}

__global__ void tp_inv_perm(const int* __restrict__ perm, int E, int* __restrict__ pos) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < E; q += gridDim.x * blockDim.x) pos[perm[q]] = q;
}

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace

int tp_csr_launch(const TPCsrArgs& a, cudaStream_t st) {
  int n = 0;
  if (!a.skip_recv) {
    cudaMemsetAsync(a.err, 0xff, sizeof(unsigned long long), st);
    if (a.E > 0) {
      tp_check<<<grid_for(a.E, 256), 256, 0, st>>>(a.sender, a.receiver, a.N, a.E, a.err);
      n++;
    }
    tp_recv_off<<<grid_for(a.N + 1, 256), 256, 0, st>>>(a.receiver, a.N, a.E, a.recv_off);
    n++;
  }
  if (a.send_off) {
    cudaMemsetAsync(a.send_cnt, 0, sizeof(int) * (a.N > 0 ? a.N : 1), st);
    if (a.E > 0) { tp_send_hist<<<grid_for(a.E, 256), 256, 0, st>>>(a.sender, a.N, a.E, a.send_cnt); n++; }
    tp_scan<<<1, 1024, 0, st>>>(a.send_cnt, a.N, a.send_off, a.send_cur);
    n++;
    if (a.E > 0) {
      tp_send_scatter<<<grid_for(a.E, 256), 256, 0, st>>>(a.sender, a.N, a.E, a.send_cur, a.send_perm);
      tp_seg_sort<<<grid_for(a.N, 128), 128, 0, st>>>(a.send_off, a.N, a.send_perm);  // (warp bitonic measured slower)
      tp_inv_perm<<<grid_for(a.E, 256), 256, 0, st>>>(a.send_perm, a.E, a.send_pos);
      n += 3;
    }
  }
  return n;
}

int tp_dh_reduce_launch(const float* dhe, const int* off, const int* perm, int N, int K, int nh, float* dh,
                        cudaStream_t st) {
  (void)perm;
  if (N <= 0) return 0;
  const bool pr = K % 2 == 0;
  const int g = grid_for((long long)N * K / (pr ? 2 : 1), 256);
#define TP_DH_CASE(NHV)                                                                  \
  case NHV:                                                                              \
    if (pr) tp_dh_reduce<2, NHV><<<g, 256, 0, st>>>(dhe, off, N, K, dh);                 \
    else tp_dh_reduce<1, NHV><<<g, 256, 0, st>>>(dhe, off, N, K, dh);                    \
    break;
  switch (nh) {
    TP_DH_CASE(1) TP_DH_CASE(2) TP_DH_CASE(3) TP_DH_CASE(4) TP_DH_CASE(5) TP_DH_CASE(6) TP_DH_CASE(7) TP_DH_CASE(8)
    TP_DH_CASE(9) TP_DH_CASE(10) TP_DH_CASE(11) TP_DH_CASE(12) TP_DH_CASE(13) TP_DH_CASE(14) TP_DH_CASE(15)
    TP_DH_CASE(16)
    default: return 0;
  }
#undef TP_DH_CASE
  return 1;
}

// dst[i] += src[i] (the sums of the TP double backward's passes, symcon_tp_backward2)
__global__ void add_inplace(float* __restrict__ dst, const float* __restrict__ src, long long n) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(dst)[i];
    const float4 b = reinterpret_cast<const float4*>(src)[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    reinterpret_cast<float4*>(dst)[i] = a;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

int add_inplace_launch(float* dst, const float* src, long long n, cudaStream_t st) {
  if (n <= 0) return 0;
  add_inplace<<<grid_for((n + 3) / 4, 256), 256, 0, st>>>(dst, src, n);
  return 1;
}

}  // namespace symcon

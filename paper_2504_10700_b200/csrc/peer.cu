// dW all-reduce over NVLink peer memory (PAPER.md:960 data-parallel all-reduce):
// every rank's dW partial lives in a symmetric buffer (torch symmetric memory). One kernel per call:
//   one-shot  (algo 1): a cross-GPU barrier on the signal pads (release/acquire at system scope),
//                       then out = sum of all ranks' partials in rank order via P2P loads;
//                       every rank reads (world-1) remote copies of the buffer.
//   two-shot  (algo 2): barrier; rank r sums slice r of every partial (rank order) and writes it
//                       in place into slice r of its own buffer (reduce-scatter); a grid-wide
//                       arrival count, then a second barrier; every rank gathers slice q from rank
//                       q's buffer (all-gather). Each rank reads 2 (world-1)/world of the buffer
//                       over NVLink instead of (world-1) times it.
// Both give bitwise the same dW on every rank (each element summed once, in rank order).
// A barrier that does not complete within spin_limit polls (~200 ns each) is a hard error: err
// is set to 1 and the block writes NaN over its part of `out` instead of any partial sum.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace symcon {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void peer_epoch_bump(unsigned* counter) { *counter += 1u; }

// thread 0 of the block waits until slot `base + p` of this rank's pad reaches `epoch` for every
// p < world; returns (block-uniform) false on timeout
__device__ bool wait_all(const PeerArgs& a, int world, int rank, int base, unsigned epoch, long long spin_limit, int* err) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    for (int p = 0; p < world && ok; p++) {
      long long spins = 0;
      while ((int)(ld_acquire_sys(a.pad[rank] + base + p) - epoch) < 0) {
        if (++spins > spin_limit) { if (err) atomicExch(err, 1); ok = 0; break; }
        __nanosleep(200);
      }
    }
  }
  __syncthreads();
  return ok != 0;
}

__device__ void nan_fill(float* out, long long lo, long long hi) {
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi; i += (long long)gridDim.x * blockDim.x)
    out[i] = __int_as_float(0x7fc00000);
}

// out[lo, hi) = sum_p src[p][lo, hi) in rank order (float4 body when lo is a multiple of 4)
__device__ void sum_range(const float* const* src, int world, long long lo, long long hi, float* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long b4 = (lo + 3) / 4, e4 = hi / 4;
  for (long long i = lo + t0; i < min(hi, 4 * b4); i += stride) {
    float s = __ldcg(src[0] + i);
    for (int p = 1; p < world; p++) s += __ldcg(src[p] + i);
    out[i] = s;
  }
  for (long long i = b4 + t0; i < e4; i += stride) {
    float4 s = __ldcg(reinterpret_cast<const float4*>(src[0]) + i);
    for (int p = 1; p < world; p++) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src[p]) + i);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
  for (long long i = max(4 * e4, 4 * b4) + t0; i < hi; i += stride) {
    float s = __ldcg(src[0] + i);
    for (int p = 1; p < world; p++) s += __ldcg(src[p] + i);
    out[i] = s;
  }
}

__device__ __forceinline__ unsigned epoch_of(unsigned epoch_host, const unsigned* epoch_dev) {
  // epoch from the host argument, or (graph-capturable form) the device counter + 1; the counter
  // is bumped by a separate one-thread kernel after this one, so every block reads the same value
  return epoch_dev ? *epoch_dev + 1u : epoch_host;
}

// rank < 0: emulation of `world` ranks on one device in one cooperative launch (rank = blockIdx.y)
__global__ void __launch_bounds__(512) peer_allreduce_1shot(PeerArgs a, int world, int rank, long long n, unsigned epoch_host,
                                                            const unsigned* epoch_dev, long long spin_limit, int* err) {
  if (rank < 0) rank = blockIdx.y;
  float* out = a.out[rank];
  const unsigned epoch = epoch_of(epoch_host, epoch_dev);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();   // this rank's partial (written by earlier kernels) visible to the peers
    for (int p = 0; p < world; p++) st_release_sys(a.pad[p] + rank, epoch);
  }
  if (!wait_all(a, world, rank, 0, epoch, spin_limit, err)) { nan_fill(out, 0, n); return; }
  sum_range(a.buf, world, 0, n, out);
}

// slice q of n floats: [q * n / world rounded to 4, ...) so slices are float4-aligned
__device__ __forceinline__ long long slice_lo(long long n, int world, int q) {
  return (q == world) ? n : ((n / 4) * q / world) * 4;
}

__global__ void __launch_bounds__(512) peer_allreduce_2shot(PeerArgs a, int world, int rank, long long n, unsigned epoch_host,
                                                            const unsigned* epoch_dev, long long spin_limit, int* err) {
  if (rank < 0) rank = blockIdx.y;
  float* out = a.out[rank];
  const unsigned epoch = epoch_of(epoch_host, epoch_dev);
  unsigned* arrive = a.pad[rank] + 2 * world;   // this rank's grid arrival counter (never read by peers)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; p++) st_release_sys(a.pad[p] + rank, epoch);
  }
  if (!wait_all(a, world, rank, 0, epoch, spin_limit, err)) { nan_fill(out, 0, n); return; }
  // reduce-scatter: slice `rank` of every partial, summed in rank order, in place into own buffer
  const long long lo = slice_lo(n, world, rank), hi = slice_lo(n, world, rank + 1);
  sum_range(a.buf, world, lo, hi, const_cast<float*>(a.buf[rank]));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    // the last block of this grid to finish its part of the slice announces it to every rank
    if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
      *arrive = 0u;
      __threadfence_system();
      for (int p = 0; p < world; p++) st_release_sys(a.pad[p] + world + rank, epoch);
    }
  }
  if (!wait_all(a, world, rank, world, epoch, spin_limit, err)) { nan_fill(out, 0, n); return; }
  // all-gather: slice q from rank q's buffer
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (int q = 0; q < world; q++) {
    const long long qlo = slice_lo(n, world, q), qhi = slice_lo(n, world, q + 1);
    const long long q4 = qlo / 4, e4 = (q == world - 1) ? n / 4 : qhi / 4;
    for (long long i = q4 + t0; i < e4; i += stride)
      reinterpret_cast<float4*>(out)[i] = __ldcg(reinterpret_cast<const float4*>(a.buf[q]) + i);
    if (q == world - 1)
      for (long long i = 4 * (n / 4) + t0; i < n; i += stride) out[i] = __ldcg(a.buf[q] + i);
  }
}

}  // namespace

int peer_allreduce_launch(const PeerArgs& a, int world, int rank, long long n, unsigned epoch, unsigned* epoch_dev,
                          int algo, long long spin_limit, int* err, int blocks, cudaStream_t st) {
  if (rank < 0) {
    // one cooperative launch over all emulated ranks: every block is resident, so blocks of
    // different ranks may wait on one another
    void* args[] = {(void*)&a, &world, &rank, &n, &epoch, &epoch_dev, &spin_limit, &err};
    const void* fn = algo == 2 ? (const void*)peer_allreduce_2shot : (const void*)peer_allreduce_1shot;
    if (cudaLaunchCooperativeKernel(fn, dim3(blocks, world), dim3(512), args, 0, st) != cudaSuccess) return -1;
  } else if (algo == 2) {
    peer_allreduce_2shot<<<blocks, 512, 0, st>>>(a, world, rank, n, epoch, epoch_dev, spin_limit, err);
  } else {
    peer_allreduce_1shot<<<blocks, 512, 0, st>>>(a, world, rank, n, epoch, epoch_dev, spin_limit, err);
  }
  if (epoch_dev) {
    peer_epoch_bump<<<1, 1, 0, st>>>(epoch_dev);
    return 2;
  }
  return 1;
}

}  // namespace symcon

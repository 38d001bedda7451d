// dW all-reduce over NVLink peer memory (PAPER.md:960 data-parallel all-reduce):
// every rank's dW partial lives in a symmetric buffer (torch symmetric memory); one kernel does a
// cross-GPU barrier on the signal pads (release/acquire at system scope) and then sums the
// partials of all ranks in rank order with P2P loads, so every rank ends with the bitwise same dW.
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

__global__ void __launch_bounds__(512) peer_allreduce(PeerArgs a, int world, int rank, long long n, unsigned epoch_host,
                                                      const unsigned* epoch_dev, float* __restrict__ out, int* err) {
  // epoch from the host argument, or (graph-capturable form) the device counter + 1; the counter
  // is bumped by a separate one-thread kernel after this one, so every block reads the same value
  const unsigned epoch = epoch_dev ? *epoch_dev + 1u : epoch_host;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();   // this rank's partial (written by earlier kernels) visible to the peers
    for (int p = 0; p < world; p++) st_release_sys(a.pad[p] + rank, epoch);
  }
  if (threadIdx.x == 0) {
    for (int p = 0; p < world; p++) {
      long long spins = 0;
      while ((int)(ld_acquire_sys(a.pad[rank] + p) - epoch) < 0) {
        if (++spins > (1ll << 24)) { atomicExch(err, 1); break; }   // ~seconds: report, never hang
        __nanosleep(200);
      }
    }
  }
  __syncthreads();
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 s = __ldcg(reinterpret_cast<const float4*>(a.buf[0]) + i);
    for (int p = 1; p < world; p++) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.buf[p]) + i);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float s = __ldcg(a.buf[0] + i);
    for (int p = 1; p < world; p++) s += __ldcg(a.buf[p] + i);
    out[i] = s;
  }
}

}  // namespace

int peer_allreduce_launch(const PeerArgs& a, int world, int rank, long long n, unsigned epoch, unsigned* epoch_dev,
                          float* out, int* err, int blocks, cudaStream_t st) {
  peer_allreduce<<<blocks, 512, 0, st>>>(a, world, rank, n, epoch, epoch_dev, out, err);
  if (epoch_dev) {
    peer_epoch_bump<<<1, 1, 0, st>>>(epoch_dev);
    return 2;
  }
  return 1;
}

}  // namespace symcon

// Shared-memory load probe for sm_100a: warp-uniform (broadcast) LDS.32/.64/.128 and per-lane
// LDS.128 throughput, in warp-instructions and delivered lane-bytes per SM clock. Tests whether a
// broadcast coefficient load costs one smem cycle per instruction or per 128 delivered bytes
// (coefficient delivery in the fwd/dA kernels).
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(512, 2) probe(float* out, int iters, long long* cyc) {
  __shared__ float4 s[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  const int lane = t & 31;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int base = (it * 16 + r) & 1023;
      if (V == 0) {        // LDS.32 broadcast
        const float* sf = reinterpret_cast<const float*>(s);
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(sf + base)));
        a0 += v;
      } else if (V == 1) { // LDS.64 broadcast
        float2 v;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(reinterpret_cast<const float2*>(s) + base)));
        a0 += v.x; a1 += v.y;
      } else if (V == 2) { // LDS.128 broadcast
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(s + base)));
        a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
      } else {             // LDS.128 per lane (conflict-free)
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(s + ((base + lane) & 1023))));
        a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
      }
    }
  }
  long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + t] = a0 + a1 + a2 + a3;
}

template <int V>
void run(const char* name, int lanebytes) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 2, threads = 512, iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  probe<V><<<blocks, threads>>>(out, 16, cyc);
  probe<V><<<blocks, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  const double instr_per_sm = 2.0 * (threads / 32) * iters * 16;  // 2 CTAs per SM
  printf("{\"probe\": \"%s\", \"warp_instr_per_sm_clk\": %.4f, \"lane_bytes_per_sm_clk\": %.1f}\n", name,
         instr_per_sm / mx, instr_per_sm * 32 * lanebytes / mx);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("lds32_broadcast", 4);
  run<1>("lds64_broadcast", 8);
  run<2>("lds128_broadcast", 16);
  run<3>("lds128_per_lane", 16);
  return 0;
}

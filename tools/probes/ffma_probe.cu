// FP32-pipe probe for sm_100a: which FFMA forms issue at full rate on B200.
// Feeds DESIGN.md's ALU roofline (the symmetric contraction is FP32-FMA bound,
// SURVEY.md §8(d)). Each variant runs one co-resident wave (148 SMs x 2 CTAs x
// 512 threads) and reports FMA lane-ops per SM clock from clock64 deltas.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
struct Coefs { float c[64]; };

__device__ __forceinline__ void fma2(float& a0, float& a1, float x0, float x1, float y0, float y1) {
  unsigned long long d, a, b, c;
  asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(y0), "f"(y1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(a0), "f"(a1));
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(d));
}

template <int V>
__global__ void __launch_bounds__(512, 2) probe(const float* __restrict__ in, float* out, int iters,
                                                Coefs cf, long long* cyc) {
  __shared__ float4 sc[256];
  int t = threadIdx.x;
  if (t < 256) sc[t] = make_float4(in[t & 63], in[(t + 1) & 63], in[(t + 2) & 63], in[(t + 3) & 63]);
  __syncthreads();
  float x[NCH], y[NCH], acc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; i++) { x[i] = in[(t + i) & 63]; y[i] = in[(t * 3 + i) & 63]; acc[i] = 0.f; }
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      if (V == 0) {  // 3 distinct register sources
#pragma unroll
        for (int i = 0; i < NCH; i++) acc[i] = fmaf(x[i], y[(i + r) & (NCH - 1)], acc[i]);
      } else if (V == 1) {  // immediate multiplier
#pragma unroll
        for (int i = 0; i < NCH; i++) acc[i] = fmaf(x[(i + r) & (NCH - 1)], 0.999f + 0.0001f * r, acc[i]);
      } else if (V == 2) {  // constant-bank multiplier (kernel param)
#pragma unroll
        for (int i = 0; i < NCH; i++) acc[i] = fmaf(x[(i + r) & (NCH - 1)], cf.c[(i * 8 + r) & 63], acc[i]);
      } else if (V == 3) {  // packed f32x2, all registers
#pragma unroll
        for (int i = 0; i < NCH; i += 2)
          fma2(acc[i], acc[i + 1], x[i], x[i + 1], y[(i + r) & (NCH - 1)], y[(i + r + 1) & (NCH - 1)]);
      } else if (V == 4) {  // broadcast LDS.128 coefficient, 4 nodes share it
#pragma unroll
        for (int i = 0; i < NCH; i += 4) {
          float4 c = sc[(it * 8 + r * 4 + i) & 255];
          acc[i] = fmaf(x[i], c.x, acc[i]); acc[i + 1] = fmaf(x[i + 1], c.x, acc[i + 1]);
          acc[i + 2] = fmaf(x[i + 2], c.x, acc[i + 2]); acc[i + 3] = fmaf(x[i + 3], c.x, acc[i + 3]);
          acc[i] = fmaf(y[i], c.y, acc[i]); acc[i + 1] = fmaf(y[i + 1], c.y, acc[i + 1]);
          acc[i + 2] = fmaf(y[i + 2], c.y, acc[i + 2]); acc[i + 3] = fmaf(y[i + 3], c.y, acc[i + 3]);
          acc[i] = fmaf(x[i+1], c.z, acc[i]); acc[i + 1] = fmaf(x[i + 2], c.z, acc[i + 1]);
          acc[i + 2] = fmaf(x[i + 3], c.z, acc[i + 2]); acc[i + 3] = fmaf(x[i], c.z, acc[i + 3]);
          acc[i] = fmaf(y[i+1], c.w, acc[i]); acc[i + 1] = fmaf(y[i + 2], c.w, acc[i + 1]);
          acc[i + 2] = fmaf(y[i + 3], c.w, acc[i + 2]); acc[i + 3] = fmaf(y[i], c.w, acc[i + 3]);
        }
      } else if (V == 5) {  // packed f32x2 with a shared (duplicated) multiplier pair
#pragma unroll
        for (int i = 0; i < NCH; i += 2)
          fma2(acc[i], acc[i + 1], x[i], x[i + 1], y[r & 7], y[r & 7]);
      } else if (V == 6) {  // multiplier shared across consecutive FFMAs (operand reuse cache)
#pragma unroll
        for (int i = 0; i < NCH; i++) acc[i] = fmaf(x[i], y[r & 7], acc[i]);
      } else if (V == 7) {  // per-lane LDS.128 coefficient (distinct address), 4 nodes share it
#pragma unroll
        for (int i = 0; i < NCH; i += 4) {
          float4 c = sc[(t + it * 8 + r * 4 + i) & 255];
          acc[i] = fmaf(x[i], c.x, acc[i]); acc[i + 1] = fmaf(x[i + 1], c.x, acc[i + 1]);
          acc[i + 2] = fmaf(x[i + 2], c.x, acc[i + 2]); acc[i + 3] = fmaf(x[i + 3], c.x, acc[i + 3]);
          acc[i] = fmaf(y[i], c.y, acc[i]); acc[i + 1] = fmaf(y[i + 1], c.y, acc[i + 1]);
          acc[i + 2] = fmaf(y[i + 2], c.y, acc[i + 2]); acc[i + 3] = fmaf(y[i + 3], c.y, acc[i + 3]);
          acc[i] = fmaf(x[i+1], c.z, acc[i]); acc[i + 1] = fmaf(x[i + 2], c.z, acc[i + 1]);
          acc[i + 2] = fmaf(x[i + 3], c.z, acc[i + 2]); acc[i + 3] = fmaf(x[i], c.z, acc[i + 3]);
          acc[i] = fmaf(y[i+1], c.w, acc[i]); acc[i + 1] = fmaf(y[i + 2], c.w, acc[i + 1]);
          acc[i + 2] = fmaf(y[i + 3], c.w, acc[i + 2]); acc[i + 3] = fmaf(y[i], c.w, acc[i + 3]);
        }
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + t] = s;
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, const float* din, float* dout, long long* dcyc, int sms, Coefs cf) {
  int iters = 4000, blocks = sms * 2, threads = 512;
  probe<V><<<blocks, threads>>>(din, dout, 10, cf, dcyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<V><<<blocks, threads>>>(din, dout, iters, cf, dcyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  static long long h[4096]; cudaMemcpy(h, dcyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0; double mean = 0; for (int b = 0; b < blocks; b++) { mx = h[b] > mx ? h[b] : mx; mean += h[b]; }
  mean /= blocks;
  double fma_per_thread = (double)iters * 8 * NCH;
  double total = fma_per_thread * threads * blocks;
  double per_sm_clk = fma_per_thread * threads * 2 / mean;
  printf("{\"variant\":\"%s\",\"ms\":%.4f,\"tfma_per_s\":%.3f,\"fma_per_sm_clk\":%.1f,\"cyc_max\":%lld,\"implied_mhz\":%.0f}\n",
         name, ms, total / ms / 1e9, per_sm_clk, mx, mean / (ms * 1e3));
}

int main() {
  int dev = 0, sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float h[64]; for (int i = 0; i < 64; i++) h[i] = 1.0f + 1e-4f * i;
  Coefs cf; for (int i = 0; i < 64; i++) cf.c[i] = 0.5f + 1e-3f * i;
  float *din, *dout; long long* dcyc;
  cudaMalloc(&din, 64 * 4); cudaMalloc(&dout, sms * 2 * 512 * 4); cudaMalloc(&dcyc, sms * 2 * 8);
  cudaMemcpy(din, h, 256, cudaMemcpyHostToDevice);
  printf("{\"sms\":%d}\n", sms);
  for (int rep = 0; rep < 2; rep++) {
    run<0>("ffma_3reg", din, dout, dcyc, sms, cf);
    run<1>("ffma_imm", din, dout, dcyc, sms, cf);
    run<2>("ffma_constbank", din, dout, dcyc, sms, cf);
    run<3>("ffma2_regs", din, dout, dcyc, sms, cf);
    run<4>("lds128_bcast_x4", din, dout, dcyc, sms, cf);
    run<5>("ffma2_shared_mul", din, dout, dcyc, sms, cf);
    run<6>("ffma_reuse_mul", din, dout, dcyc, sms, cf);
    run<7>("lds128_perlane_x4", din, dout, dcyc, sms, cf);
  }
  cudaError_t e = cudaGetLastError(); printf("{\"err\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}

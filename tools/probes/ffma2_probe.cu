// FP32-pipe probe v2 for sm_100a: issue rate of the FFMA2 / FFMA operand forms the
// generated kernels use. Fixes r01's accounting: per SM, cycles =
// max(end) - min(start) over the CTAs that ran on that SM (%smid, clock64), lane-ops = the sum of
// those CTAs' lane-ops; reported as lane-ops per SM clock (peak 128) and as a fraction of 128.
// Every variant runs exactly one co-resident wave (148 SMs x OCC CTAs x 256 threads), 16
// independent accumulator chains per thread (latency hidden).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 bc(float s) { return pk(s, s); }

#define NA 16
struct Rec { long long t0, t1; int smid; };

template <int V>
__global__ void __launch_bounds__(256) probe(const float* __restrict__ in, float* out, int iters, Rec* rec) {
  const int t = threadIdx.x;
  u64 x[NA], y[NA], acc[NA];
  float s[NA];
#pragma unroll
  for (int i = 0; i < NA; i++) {
    x[i] = pk(in[(t + i) & 63], in[(t + 2 * i + 1) & 63]);
    y[i] = pk(in[(3 * t + i) & 63], in[(t + 5 * i + 2) & 63]);
    s[i] = in[(7 * t + i) & 63];
    acc[i] = pk(0.f, 0.f);
  }
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
#pragma unroll
      for (int i = 0; i < NA; i++) {
        const int j = (i + r) & (NA - 1);
        if (V == 0) acc[i] = fma2(x[j], bc(s[j]), acc[i]);           // pair x scalar + acc (the fwd/dW form)
        if (V == 1) acc[i] = fma2(x[j], y[(j + 3) & (NA - 1)], acc[i]); // three distinct pairs
        if (V == 2) acc[i] = fma2(x[j], y[r], acc[i]);                 // second pair shared by 16 consecutive
        if (V == 3) acc[i] = fma2(y[r], x[j], acc[i]);                 // first pair shared by 16 consecutive
        if (V == 4) acc[i] = fma2(x[j], bc(s[r]), acc[i]);             // scalar shared by 16 consecutive
        if (V == 5) acc[i] = mul2(x[j], acc[i]);                       // FMUL2 two pairs
        if (V == 6) acc[i] = fma2(x[j], bc(0.999f), acc[i]);           // constant multiplier
        if (V == 7) {                                                  // scalar FFMA, 3 regs (halves)
          float a0 = lo(acc[i]), a1 = hi(acc[i]);
          a0 = fmaf(lo(x[j]), s[(j + 1) & (NA - 1)], a0);
          a1 = fmaf(hi(x[j]), s[(j + 2) & (NA - 1)], a1);
          acc[i] = pk(a0, a1);
        }
        if (V == 8) acc[i] = fma2(x[i], bc(s[r]), acc[i]);             // scalar shared, x per accumulator
        if (V == 9) {                                                  // Horner-like: inner = sum c A (scalar), then 3-pair
          acc[i] = fma2(x[j], bc(s[j]), acc[i]);
          if ((i & 3) == 3) y[r] = fma2(acc[i], x[(j + 7) & (NA - 1)], y[r]);
        }
      }
    }
  }
  long long t1 = clock64();
  u64 sum = pk(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < NA; i++) sum = fma2(acc[i], y[i & 3], sum);
  out[blockIdx.x * blockDim.x + t] = lo(sum) + hi(sum);
  if (t == 0) rec[blockIdx.x] = {t0, t1, (int)smid};
}

template <int V>
void run(const char* name, double ops_per_inner, const float* din, float* dout, Rec* drec, int sms, int occ) {
  const int iters = 2000, blocks = sms * occ, threads = 256;
  probe<V><<<blocks, threads>>>(din, dout, 10, drec);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<V><<<blocks, threads>>>(din, dout, iters, drec);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<Rec> h(blocks);
  cudaMemcpy(h.data(), drec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost);
  // per SM: lane-ops of its CTAs / (last end - first start)
  std::vector<long long> mn(sms, (1ll << 62)), mx(sms, 0);
  std::vector<int> cnt(sms, 0);
  for (auto& r : h) { if (r.smid < 0 || r.smid >= sms) continue; mn[r.smid] = std::min(mn[r.smid], r.t0); mx[r.smid] = std::max(mx[r.smid], r.t1); cnt[r.smid]++; }
  const double lane_ops_per_cta = (double)iters * 4 * ops_per_inner * threads;
  std::vector<double> per;
  for (int q = 0; q < sms; q++) if (cnt[q]) per.push_back(lane_ops_per_cta * cnt[q] / (double)(mx[q] - mn[q]));
  std::sort(per.begin(), per.end());
  const double med = per.empty() ? 0 : per[per.size() / 2];
  const double total = lane_ops_per_cta * blocks;
  printf("{\"variant\":\"%s\",\"occ_ctas_per_sm\":%d,\"ms\":%.4f,\"t_lane_ops_per_s\":%.3f,\"lane_ops_per_sm_clk_median\":%.1f,"
         "\"frac_of_128\":%.3f,\"implied_mhz\":%.0f}\n",
         name, occ, ms, total / ms / 1e9, med, med / 128.0, total / (ms * 1e-3) / (med * sms) / 1e6);
}

int main() {
  int dev = 0, sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float h[64]; for (int i = 0; i < 64; i++) h[i] = 1.0f + 1e-4f * i;
  float *din, *dout; Rec* drec;
  cudaMalloc(&din, 64 * 4); cudaMalloc(&dout, sms * 8 * 256 * 4); cudaMalloc(&drec, sms * 8 * sizeof(Rec));
  cudaMemcpy(din, h, 256, cudaMemcpyHostToDevice);
  printf("{\"sms\":%d}\n", sms);
  for (int occ : {2, 4}) {
    // lane-ops per inner iteration (16 instructions; FFMA2 = 2 lane-ops)
    run<0>("ffma2_pair_x_scalar", 32, din, dout, drec, sms, occ);
    run<1>("ffma2_three_pairs", 32, din, dout, drec, sms, occ);
    run<2>("ffma2_second_pair_shared", 32, din, dout, drec, sms, occ);
    run<3>("ffma2_first_pair_shared", 32, din, dout, drec, sms, occ);
    run<4>("ffma2_scalar_shared", 32, din, dout, drec, sms, occ);
    run<5>("fmul2_two_pairs", 32, din, dout, drec, sms, occ);
    run<6>("ffma2_const_mul", 32, din, dout, drec, sms, occ);
    run<7>("ffma_scalar_3reg_x2", 32, din, dout, drec, sms, occ);
    run<8>("ffma2_scalar_shared_x_per_acc", 32, din, dout, drec, sms, occ);
    run<9>("ffma2_horner_mix_4to1", 40, din, dout, drec, sms, occ);
  }
  cudaError_t e = cudaGetLastError(); printf("{\"err\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}

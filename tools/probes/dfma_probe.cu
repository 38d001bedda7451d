// FP64-pipe probe for sm_100a (the fp64 roofline): issue rate of scalar DFMA in the
// operand forms the plain scalar kernels use (codegen_simple.cpp). Same accounting as ffma2_probe.cu:
// per SM, cycles = max(end) - min(start) over the CTAs that ran on that SM (%smid, clock64); one
// co-resident wave (148 SMs x OCC CTAs x 256 threads), 16 independent accumulator chains per thread.
// Reported as DFMA lane-ops per SM clock and T lane-ops/s at the measured clock.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define NA 16
struct Rec { long long t0, t1; int smid; };

template <int V>
__global__ void __launch_bounds__(256) probe(const double* __restrict__ in, double* out, int iters, Rec* rec) {
  const int t = threadIdx.x;
  double x[NA], s[NA], acc[NA];
#pragma unroll
  for (int i = 0; i < NA; i++) {
    x[i] = in[(t + i) & 63];
    s[i] = in[(7 * t + i) & 63];
    acc[i] = 0.0;
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
        if (V == 0) acc[i] = fma(x[j], s[(j + 1) & (NA - 1)], acc[i]);   // three registers
        if (V == 1) acc[i] = fma(x[j], s[r], acc[i]);                    // multiplier shared by 16 consecutive
        if (V == 2) acc[i] = fma(x[j], 0.999, acc[i]);                   // constant multiplier
      }
    }
  }
  long long t1 = clock64();
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < NA; i++) sum += acc[i];
  out[blockIdx.x * blockDim.x + t] = sum;
  if (t == 0) rec[blockIdx.x] = {t0, t1, (int)smid};
}

template <int V>
void run(const char* name, const double* din, double* dout, Rec* drec, int sms, int occ) {
  const int iters = 500, blocks = sms * occ, threads = 256;
  probe<V><<<blocks, threads>>>(din, dout, 10, drec);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<V><<<blocks, threads>>>(din, dout, iters, drec);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<Rec> h(blocks);
  cudaMemcpy(h.data(), drec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost);
  std::vector<long long> mn(sms, (1ll << 62)), mx(sms, 0);
  std::vector<int> cnt(sms, 0);
  for (auto& r : h) { if (r.smid < 0 || r.smid >= sms) continue; mn[r.smid] = std::min(mn[r.smid], r.t0); mx[r.smid] = std::max(mx[r.smid], r.t1); cnt[r.smid]++; }
  const double lane_ops_per_cta = (double)iters * 4 * NA * threads;
  std::vector<double> per;
  for (int q = 0; q < sms; q++) if (cnt[q]) per.push_back(lane_ops_per_cta * cnt[q] / (double)(mx[q] - mn[q]));
  std::sort(per.begin(), per.end());
  const double med = per.empty() ? 0 : per[per.size() / 2];
  const double total = lane_ops_per_cta * blocks;
  printf("{\"variant\":\"%s\",\"occ_ctas_per_sm\":%d,\"ms\":%.4f,\"t_dfma_lane_ops_per_s\":%.3f,\"dfma_per_sm_clk_median\":%.2f,"
         "\"implied_mhz\":%.0f}\n",
         name, occ, ms, total / ms / 1e9, med, total / (ms * 1e-3) / (med * sms) / 1e6);
}

int main() {
  int dev = 0, sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double h[64]; for (int i = 0; i < 64; i++) h[i] = 1.0 + 1e-4 * i;
  double *din, *dout; Rec* drec;
  cudaMalloc(&din, 64 * 8); cudaMalloc(&dout, sms * 8 * 256 * 8); cudaMalloc(&drec, sms * 8 * sizeof(Rec));
  cudaMemcpy(din, h, 64 * 8, cudaMemcpyHostToDevice);
  printf("{\"sms\":%d}\n", sms);
  for (int occ : {2, 4}) {
    run<0>("dfma_three_regs", din, dout, drec, sms, occ);
    run<1>("dfma_shared_multiplier", din, dout, drec, sms, occ);
    run<2>("dfma_const_multiplier", din, dout, drec, sms, occ);
  }
  cudaError_t e = cudaGetLastError(); printf("{\"err\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}

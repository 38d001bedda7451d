// Element bucketing: a stable counting sort of nodes by element so
// that every 64-node tile of the contraction kernels belongs to ONE element (W depends on
// z_i) and its per-(element, channel) coefficients are warp-uniform.
//
//   bk_hist     per 1024-node chunk: histogram over E+1 buckets (bucket E = out-of-range
//               node_elem; the first such node index is recorded in *err)
//   bk_scan     one CTA: chunk offsets (element-major), seg_off, the tile list (<= 64 nodes,
//               one element each) and the dW item list (<= R tiles of one element each)
//   bk_scatter  one warp per chunk, 32 nodes at a time with __match_any_sync ranks: stable
//   bk_fill_nan writes NaN rows for nodes in the out-of-range bucket
// All integer work; deterministic for a given node_elem.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace symcon {

static constexpr int kChunk = 1024;

__global__ void bk_hist(const int* __restrict__ ne, int N, int E, int* __restrict__ hist,
                        int* __restrict__ chunk_bad) {
  extern __shared__ int h[];
  __shared__ int bad;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) h[e] = 0;
  if (threadIdx.x == 0) bad = 0x7fffffff;
  __syncthreads();
  const int base = blockIdx.x * kChunk;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    int i = base + t;
    if (i >= N) break;
    int e = ne[i];
    if (e < 0 || e >= E) {
      e = E;
      atomicMin(&bad, i);
    }
    atomicAdd(&h[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += blockDim.x) hist[(size_t)blockIdx.x * (E + 1) + e] = h[e];
  if (threadIdx.x == 0) chunk_bad[blockIdx.x] = bad;
}

__global__ void __launch_bounds__(1024) bk_scan(const int* __restrict__ hist, int nchunks, int E, int* __restrict__ off,
                        int* __restrict__ seg_off, int4* __restrict__ tiles, int* __restrict__ n_tiles,
                        int4* __restrict__ items, int* __restrict__ n_items, int* __restrict__ item_off,
                        int* __restrict__ tile_off, int* __restrict__ tile_perm, int tile_nodes, int tiles_per_item,
                        const int* __restrict__ chunk_bad, unsigned long long* __restrict__ err,
                        int* __restrict__ zero_buf, int zero_n) {
  extern __shared__ int sm[];   // tot[E+1], tile_off[E+1], itm_off[E+1]
  int* tot = sm;
  int* toff = sm + (E + 1);
  int* ioff = sm + 2 * (E + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5, E1 = E + 1;
  for (int e = tid; e <= E; e += blockDim.x) tot[e] = 0;
  if (zero_buf)
    for (int x = tid; x < zero_n; x += blockDim.x) zero_buf[x] = 0;
  __syncthreads();
  // 1. element totals: coalesced pass over the [chunk][E+1] histogram with smem atomics
  for (int x = tid; x < nchunks * E1; x += blockDim.x) {
    const int h = hist[x];
    if (h) atomicAdd(&tot[x % E1], h);
  }
  __shared__ int bad;
  if (tid == 0) bad = 0x7fffffff;
  __syncthreads();
  for (int c = tid; c < nchunks; c += blockDim.x) atomicMin(&bad, chunk_bad[c]);
  __syncthreads();
  if (tid == 0) *err = (bad == 0x7fffffff) ? ~0ull : (unsigned long long)bad;
  // 2. segment / tile / item offsets: block-wide exclusive scans of (count, tiles, items) per element
  if (E1 <= (int)blockDim.x) {
    __shared__ int wsum[3][32];
    int c = 0, nt = 0, ni = 0;
    if (tid < E1) {
      c = tot[tid];
      nt = (tid < E) ? (c + tile_nodes - 1) / tile_nodes : 0;
      ni = (nt + tiles_per_item - 1) / tiles_per_item;
    }
    int xc = c, xt = nt, xi = ni;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yc = __shfl_up_sync(0xffffffffu, xc, o), yt = __shfl_up_sync(0xffffffffu, xt, o),
                yi = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) { xc += yc; xt += yt; xi += yi; }
    }
    if (lane == 31) { wsum[0][warp] = xc; wsum[1][warp] = xt; wsum[2][warp] = xi; }
    __syncthreads();
    if (warp == 0) {
      int a = wsum[0][lane], b = wsum[1][lane], d = wsum[2][lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o),
                  yd = __shfl_up_sync(0xffffffffu, d, o);
        if (lane >= o) { a += ya; b += yb; d += yd; }
      }
      wsum[0][lane] = a; wsum[1][lane] = b; wsum[2][lane] = d;  // inclusive warp totals
    }
    __syncthreads();
    const int bc = warp ? wsum[0][warp - 1] : 0, bt = warp ? wsum[1][warp - 1] : 0, bi = warp ? wsum[2][warp - 1] : 0;
    __syncthreads();
    if (tid < E1) {
      const int sc = bc + xc - c, st2 = bt + xt - nt, si = bi + xi - ni;  // exclusive
      tot[tid] = sc; seg_off[tid] = sc;
      toff[tid] = st2; tile_off[tid] = st2;
      ioff[tid] = si; item_off[tid] = si;
      if (tid == E) {
        seg_off[E + 1] = sc + c;
        tile_off[E] = st2;     // bucket E has no tiles
        *n_tiles = st2;
        *n_items = si;
        item_off[E + 1] = si;
      }
    }
  } else if (tid == 0) {
    int s = 0, ts = 0, is = 0;
    for (int e = 0; e <= E; e++) {
      int c = tot[e];
      tot[e] = s;
      seg_off[e] = s;
      s += c;
      int nt = (e < E) ? (c + tile_nodes - 1) / tile_nodes : 0;
      toff[e] = ts;
      tile_off[e] = ts;
      ts += nt;
      int ni = (nt + tiles_per_item - 1) / tiles_per_item;
      ioff[e] = is;
      item_off[e] = is;
      is += ni;
    }
    seg_off[E + 1] = s;
    tile_off[E] = ts;
    *n_tiles = ts;
    *n_items = is;
    item_off[E + 1] = is;
  }
  __syncthreads();
  // 3. per element (one warp each): exclusive scan over chunks -> off[c][e]; tiles, items, padding
  for (int e = warp; e <= E; e += nw) {
    int run = tot[e];
    for (int c0 = 0; c0 < nchunks; c0 += 32) {
      const int c = c0 + lane;
      const int h = (c < nchunks) ? hist[(size_t)c * E1 + e] : 0;
      int x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (c < nchunks) off[(size_t)c * E1 + e] = run + x - h;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (e < E) {
      const int start = tot[e], cnt = run - tot[e];
      const int nt = (cnt + tile_nodes - 1) / tile_nodes;
      for (int t = lane; t < nt; t += 32) {
        const int c0 = t * tile_nodes;
        tiles[toff[e] + t] = make_int4(e, start + c0, min(tile_nodes, cnt - c0), t);
      }
      const int ni = (nt + tiles_per_item - 1) / tiles_per_item;
      for (int q = lane; q < ni; q += 32) {
        const int t0 = q * tiles_per_item;
        items[ioff[e] + q] = make_int4(e, toff[e] + t0, min(tiles_per_item, nt - t0), q);
      }
      if (nt > 0)  // empty slots of the element's last tile (the scatter fills the others)
        for (int q = cnt - (nt - 1) * tile_nodes + lane; q < tile_nodes; q += 32)
          tile_perm[(size_t)(toff[e] + nt - 1) * tile_nodes + q] = -1;
    }
  }
}

__global__ void bk_scatter(const int* __restrict__ ne, int N, int E, const int* __restrict__ off,
                           const int* __restrict__ seg_off, const int* __restrict__ tile_off, int tile_nodes,
                           int* __restrict__ perm, int* __restrict__ tile_perm) {
  extern __shared__ int cnt[];
  const int lane = threadIdx.x;
  for (int e = lane; e <= E; e += 32) cnt[e] = off[(size_t)blockIdx.x * (E + 1) + e];
  __syncwarp();
  const int base = blockIdx.x * kChunk;
  int ev[kChunk / 32];  // all 32 groups' elements in flight at once (latency hiding)
#pragma unroll
  for (int g = 0; g < kChunk / 32; g++) {
    const int i = base + g * 32 + lane;
    int e = -1;
    if (i < N) {
      e = ne[i];
      if (e < 0 || e >= E) e = E;
    }
    ev[g] = e;
  }
#pragma unroll
  for (int g = 0; g < kChunk / 32; g++) {
    const int i = base + g * 32 + lane;
    const int e = ev[g];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    const int leader = __ffs(peers) - 1;
    int pos = 0;
    if (e >= 0) pos = cnt[e] + rank;
    __syncwarp();
    if (e >= 0 && lane == leader) cnt[e] += __popc(peers);
    __syncwarp();
    if (e >= 0) perm[pos] = i;
    if (e >= 0 && e < E) {  // padded per-tile node list: tile_perm[tile][slot], -1 = empty slot
      const int r = pos - seg_off[e];
      tile_perm[(size_t)(tile_off[e] + r / tile_nodes) * tile_nodes + r % tile_nodes] = i;
    }
  }
}

// Block-parallel stable scatter for E + 1 <= kWarpE: one CTA (32 warps) per 1024-node chunk.
// Warp w ranks its 32 nodes with one __match_any_sync; per-warp element counts go to smem,
// an exclusive scan over warps (per element) gives each warp's base; stable by construction.
static constexpr int kWarpE = 512;
__global__ void __launch_bounds__(1024) bk_scatter_blk(const int* __restrict__ ne, int N, int E, const int* __restrict__ off,
                                                       const int* __restrict__ seg_off, const int* __restrict__ tile_off,
                                                       int tile_nodes, int* __restrict__ perm, int* __restrict__ tile_perm) {
  extern __shared__ int cw[];  // [32 warps][E+1]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, E1 = E + 1;
  for (int x = tid; x < 32 * E1; x += 1024) cw[x] = 0;
  __syncthreads();
  const int i = blockIdx.x * kChunk + tid;
  int e = -1;
  if (i < N) {
    e = ne[i];
    if (e < 0 || e >= E) e = E;
  }
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  if (e >= 0 && lane == __ffs(peers) - 1) cw[warp * E1 + e] = __popc(peers);
  __syncthreads();
  // exclusive scan over warps for each element, seeded with the chunk offset
  for (int x = tid; x < E1; x += 1024) {
    int r = off[(size_t)blockIdx.x * E1 + x];
#pragma unroll 8
    for (int w = 0; w < 32; w++) {
      const int c = cw[w * E1 + x];
      cw[w * E1 + x] = r;
      r += c;
    }
  }
  __syncthreads();
  if (e >= 0) {
    const int pos = cw[warp * E1 + e] + rank;
    perm[pos] = i;
    if (e < E) {
      const int r = pos - seg_off[e];
      tile_perm[(size_t)(tile_off[e] + r / tile_nodes) * tile_nodes + r % tile_nodes] = i;
    }
  }
}

__global__ void bk_fill_nan(const int* __restrict__ perm, const int* __restrict__ seg_off, int E,
                            float* __restrict__ out, long long row) {
  const int s = seg_off[E], t = seg_off[E + 1];
  const float nan = __int_as_float(0x7fc00000);
  for (int q = s + blockIdx.x; q < t; q += gridDim.x) {
    float* r = out + (long long)perm[q] * row;
    for (long long x = threadIdx.x; x < row; x += blockDim.x) r[x] = nan;
  }
}

// One cooperative launch for the whole bucketing (E + 1 <= kWarpE): CTA b owns 1024-node chunks
// [b*S, (b+1)*S). Phase 1: per-chunk histograms -> hist. grid sync. Phase 2: every CTA derives the
// element totals, seg_off and its own chunks' offsets from hist (no second sync); CTA 0 also writes
// seg_off, the tile / item lists, tile_off / item_off, the padding of tile_perm, the error word and
// zeroes zero_buf. Phase 3: the block-parallel stable scatter of bk_scatter_blk on each own chunk.
// Same results as bk_hist + bk_scan + bk_scatter_blk (deterministic, stable).
__global__ void __launch_bounds__(1024) bk_fused(BucketArgs a, int nchunks, int S) {
  namespace cg = cooperative_groups;
  extern __shared__ int sm[];   // h[E+1] | tot[E+1] | base[E+1] | cw[32][E+1]
  const int E = a.E, E1 = E + 1, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int* h = sm;
  int* tot = sm + E1;
  int* base = sm + 2 * E1;
  int* cw = sm + 3 * E1;
  __shared__ int bad;
  const int c0 = blockIdx.x * S, c1 = min(nchunks, c0 + S);
  // ---- phase 1: histograms of the own chunks
  for (int c = c0; c < c1; c++) {
    for (int e = tid; e <= E; e += blockDim.x) h[e] = 0;
    if (tid == 0) bad = 0x7fffffff;
    __syncthreads();
    const int i = c * 1024 + tid;
    if (i < a.N) {
      int e = a.node_elem[i];
      if (e < 0 || e >= E) { e = E; atomicMin(&bad, i); }
      atomicAdd(&h[e], 1);
    }
    __syncthreads();
    for (int e = tid; e <= E; e += blockDim.x) a.hist[(size_t)c * E1 + e] = h[e];
    if (tid == 0) a.chunk_bad[c] = bad;
    __syncthreads();
  }
  cg::this_grid().sync();
  // ---- phase 2: totals, element offsets (exclusive scan), this CTA's first chunk offset per element
  for (int e = tid; e <= E; e += blockDim.x) {
    int t = 0, b = 0;
    for (int c = 0; c < nchunks; c++) {
      const int v = __ldcg(a.hist + (size_t)c * E1 + e);
      if (c < c0) b += v;
      t += v;
    }
    tot[e] = t;
    base[e] = b;
  }
  __syncthreads();
  if (tid == 0) {   // exclusive scan of totals (E1 <= 512: serial is short)
    int run = 0;
    for (int e = 0; e <= E; e++) { const int t = tot[e]; tot[e] = run; run += t; }
  }
  __syncthreads();
  // tot[e] now = seg_off[e]
  if (blockIdx.x == 0) {
    if (tid == 0) {
      int b = 0x7fffffff;
      for (int c = 0; c < nchunks; c++) b = min(b, __ldcg(a.chunk_bad + c));
      *a.err = (b == 0x7fffffff) ? ~0ull : (unsigned long long)b;
      int ts = 0, is = 0;
      for (int e = 0; e <= E; e++) {
        const int cnt = (e < E ? tot[e + 1] : a.N) - tot[e];
        a.seg_off[e] = tot[e];
        const int nt = (e < E) ? (cnt + a.tile_nodes - 1) / a.tile_nodes : 0;
        a.tile_off[e] = ts;
        a.item_off[e] = is;
        ts += nt;
        is += (nt + a.tiles_per_item - 1) / a.tiles_per_item;
      }
      a.seg_off[E + 1] = a.N;
      *a.n_tiles = ts;
      *a.n_items = is;
      a.item_off[E + 1] = is;
    }
    if (a.zero_buf)
      for (int x = tid; x < a.zero_n; x += blockDim.x) a.zero_buf[x] = 0;
    __syncthreads();
    // tiles / items / padding, one warp per element (as bk_scan step 3)
    for (int e = warp; e < E; e += blockDim.x >> 5) {
      const int start = tot[e], cnt = tot[e + 1] - tot[e];
      const int nt = (cnt + a.tile_nodes - 1) / a.tile_nodes, toff = a.tile_off[e], ioff = a.item_off[e];
      for (int t = lane; t < nt; t += 32) {
        const int q0 = t * a.tile_nodes;
        a.tiles[toff + t] = make_int4(e, start + q0, min(a.tile_nodes, cnt - q0), t);
      }
      const int ni = (nt + a.tiles_per_item - 1) / a.tiles_per_item;
      for (int q = lane; q < ni; q += 32) {
        const int t0 = q * a.tiles_per_item;
        a.items[ioff + q] = make_int4(e, toff + t0, min(a.tiles_per_item, nt - t0), q);
      }
      if (nt > 0)
        for (int q = cnt - (nt - 1) * a.tile_nodes + lane; q < a.tile_nodes; q += 32)
          a.tile_perm[(size_t)(toff + nt - 1) * a.tile_nodes + q] = -1;
    }
  }
  // per-element tile offsets for the scatter (every CTA; same arithmetic as CTA 0's list)
  __syncthreads();
  if (tid == 0) {
    int ts = 0;
    for (int e = 0; e <= E; e++) {
      const int cnt = (e < E ? tot[e + 1] : a.N) - tot[e];
      h[e] = ts;   // tile_off (h reused)
      ts += (e < E) ? (cnt + a.tile_nodes - 1) / a.tile_nodes : 0;
    }
  }
  __syncthreads();
  // ---- phase 3: stable scatter of the own chunks (bk_scatter_blk)
  for (int c = c0; c < c1; c++) {
    for (int x = tid; x < 32 * E1; x += blockDim.x) cw[x] = 0;
    __syncthreads();
    const int i = c * 1024 + tid;
    int e = -1;
    if (i < a.N) {
      e = a.node_elem[i];
      if (e < 0 || e >= E) e = E;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (e >= 0 && lane == __ffs(peers) - 1) cw[warp * E1 + e] = __popc(peers);
    __syncthreads();
    for (int x = tid; x < E1; x += blockDim.x) {
      int r = tot[x] + base[x];
      base[x] += __ldcg(a.hist + (size_t)c * E1 + x);   // next own chunk starts after this one
#pragma unroll 8
      for (int w = 0; w < 32; w++) {
        const int v = cw[w * E1 + x];
        cw[w * E1 + x] = r;
        r += v;
      }
    }
    __syncthreads();
    if (e >= 0) {
      const int pos = cw[warp * E1 + e] + rank;
      a.perm[pos] = i;
      if (e < E) {
        const int r = pos - tot[e];
        a.tile_perm[(size_t)(h[e] + r / a.tile_nodes) * a.tile_nodes + r % a.tile_nodes] = i;
      }
    }
    __syncthreads();
  }
}

int bucket_launch(const BucketArgs& a, cudaStream_t st) {
  const int nchunks = (a.N + kChunk - 1) / kChunk;
  if (a.fused && a.N > 0 && a.E + 1 <= kWarpE) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int S = (nchunks + sms - 1) / sms, nb = (nchunks + S - 1) / S;
    const size_t smem = sizeof(int) * 35 * (size_t)(a.E + 1);
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(bk_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024); attr = true; }
    BucketArgs aa = a;
    int nc = nchunks, ss = S;
    void* args[] = {&aa, &nc, &ss};
    if (cudaLaunchCooperativeKernel((const void*)bk_fused, dim3(nb), dim3(1024), args, smem, st) == cudaSuccess) return 1;
    cudaGetLastError();   // fall back to the three kernels
  }
  const size_t sm_e = sizeof(int) * (a.E + 1);
  if (a.N > 0) bk_hist<<<nchunks, 256, sm_e, st>>>(a.node_elem, a.N, a.E, a.hist, a.chunk_bad);
  if (3 * sm_e > 48 * 1024) cudaFuncSetAttribute(bk_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * sm_e));
  bk_scan<<<1, 1024, 3 * sm_e, st>>>(a.hist, nchunks, a.E, a.off, a.seg_off, a.tiles, a.n_tiles, a.items,
                                    a.n_items, a.item_off, a.tile_off, a.tile_perm, a.tile_nodes, a.tiles_per_item,
                                    a.chunk_bad, a.err, a.zero_buf, a.zero_n);
  if (a.N > 0) {
    if (a.E + 1 <= kWarpE && 32 * sm_e > 48 * 1024)
      cudaFuncSetAttribute(bk_scatter_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(32 * sm_e));
    if (a.E + 1 <= kWarpE)
      bk_scatter_blk<<<nchunks, 1024, 32 * sm_e, st>>>(a.node_elem, a.N, a.E, a.off, a.seg_off, a.tile_off, a.tile_nodes,
                                                       a.perm, a.tile_perm);
    else
      bk_scatter<<<nchunks, 32, sm_e, st>>>(a.node_elem, a.N, a.E, a.off, a.seg_off, a.tile_off, a.tile_nodes, a.perm,
                                            a.tile_perm);
  }
  return a.N > 0 ? 3 : 1;
}

int fill_nan_launch(const int* perm, const int* seg_off, int E, float* out, long long row, cudaStream_t st) {
  bk_fill_nan<<<64, 128, 0, st>>>(perm, seg_off, E, out, row);
  return 1;
}

// Fixed-order segmented sum of the dW S partials over each element's items (the items of an
// element are contiguous). One thread per (z, j, k); 4-way unrolled loads for memory parallelism,
// summed in item order so the result is bitwise deterministic.
__global__ void dw_reduce_items(const float* __restrict__ spart, const int* __restrict__ item_off, int npad, int K,
                                float* __restrict__ stot, int ppi) {
  // ppi < 0: single-item elements were written straight into stot by the dW kernel (skip them)
  const bool skip_single = ppi < 0;
  if (skip_single) ppi = 1;
  const int z = blockIdx.y;
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)npad * K;
  if (slot >= per) return;
  const int it0 = item_off[z] * ppi, it1 = item_off[z + 1] * ppi;   // ppi partials per item, in order
  if (skip_single && it1 - it0 == 1) return;
  // 8 independent partial sums (loads in flight together), combined in a fixed order
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int it = it0;
  for (; it + 8 <= it1; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; u++) a[u] += spart[(it + u) * per + slot];
  }
  for (int u = 0; it < it1; it++, u++) a[u] += spart[it * per + slot];
  const float s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  stot[(long long)z * per + slot] = s;
}

int reduce_items_launch(const float* spart, const int* item_off, int E, int npad, int K, float* stot, cudaStream_t st,
                        int parts_per_item) {
  const long long per = (long long)npad * K;
  dim3 grid((unsigned)((per + 255) / 256), E);
  dw_reduce_items<<<grid, 256, 0, st>>>(spart, item_off, npad, K, stot, parts_per_item);
  return 1;
}

size_t bucket_chunks(int64_t N) { return (size_t)((N + kChunk - 1) / kChunk); }

}  // namespace symcon

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

__global__ void bk_scan(const int* __restrict__ hist, int nchunks, int E, int* __restrict__ off,
                        int* __restrict__ seg_off, int4* __restrict__ tiles, int* __restrict__ n_tiles,
                        int4* __restrict__ items, int* __restrict__ n_items, int* __restrict__ item_off,
                        int* __restrict__ tile_off, int* __restrict__ tile_perm, int tile_nodes, int tiles_per_item,
                        const int* __restrict__ chunk_bad, unsigned long long* __restrict__ err) {
  extern __shared__ int sm[];   // tot[E+1], tile_off[E+1], itm_off[E+1]
  int* tot = sm;
  int* toff = sm + (E + 1);
  int* ioff = sm + 2 * (E + 1);
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    int s = 0;
#pragma unroll 8
    for (int c = 0; c < nchunks; c++) s += hist[(size_t)c * (E + 1) + e];
    tot[e] = s;
  }
  if (threadIdx.x == 0) {
    int b = 0x7fffffff;
    for (int c = 0; c < nchunks; c++) b = min(b, chunk_bad[c]);
    *err = (b == 0x7fffffff) ? ~0ull : (unsigned long long)b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0, ts = 0, is = 0;
    for (int e = 0; e <= E; e++) {
      int c = tot[e];
      tot[e] = s;          // becomes the segment start
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
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    int r = tot[e];
#pragma unroll 8
    for (int c = 0; c < nchunks; c++) {
      off[(size_t)c * (E + 1) + e] = r;
      r += hist[(size_t)c * (E + 1) + e];
    }
    if (e < E) {
      const int start = tot[e], cnt = r - tot[e];
      const int nt = (cnt + tile_nodes - 1) / tile_nodes;
      for (int t = 0; t < nt; t++) {
        int c0 = t * tile_nodes;
        int c = min(tile_nodes, cnt - c0);
        tiles[toff[e] + t] = make_int4(e, start + c0, c, t);
      }
      if (nt > 0)  // empty slots of the element's last tile (the scatter fills the others)
        for (int q = cnt - (nt - 1) * tile_nodes; q < tile_nodes; q++) tile_perm[(size_t)(toff[e] + nt - 1) * tile_nodes + q] = -1;
      const int ni = (nt + tiles_per_item - 1) / tiles_per_item;
      for (int q = 0; q < ni; q++) {
        int t0 = q * tiles_per_item;
        items[ioff[e] + q] = make_int4(e, toff[e] + t0, min(tiles_per_item, nt - t0), q);
      }
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

__global__ void bk_fill_nan(const int* __restrict__ perm, const int* __restrict__ seg_off, int E,
                            float* __restrict__ out, long long row) {
  const int s = seg_off[E], t = seg_off[E + 1];
  const float nan = __int_as_float(0x7fc00000);
  for (int q = s + blockIdx.x; q < t; q += gridDim.x) {
    float* r = out + (long long)perm[q] * row;
    for (long long x = threadIdx.x; x < row; x += blockDim.x) r[x] = nan;
  }
}

int bucket_launch(const BucketArgs& a, cudaStream_t st) {
  const int nchunks = (a.N + kChunk - 1) / kChunk;
  const size_t sm_e = sizeof(int) * (a.E + 1);
  if (a.N > 0) bk_hist<<<nchunks, 256, sm_e, st>>>(a.node_elem, a.N, a.E, a.hist, a.chunk_bad);
  bk_scan<<<1, 256, 3 * sm_e, st>>>(a.hist, nchunks, a.E, a.off, a.seg_off, a.tiles, a.n_tiles, a.items,
                                    a.n_items, a.item_off, a.tile_off, a.tile_perm, a.tile_nodes, a.tiles_per_item,
                                    a.chunk_bad, a.err);
  if (a.N > 0)
    bk_scatter<<<nchunks, 32, sm_e, st>>>(a.node_elem, a.N, a.E, a.off, a.seg_off, a.tile_off, a.tile_nodes, a.perm,
                                          a.tile_perm);
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
                                float* __restrict__ stot) {
  const int z = blockIdx.y;
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)npad * K;
  if (slot >= per) return;
  const int it0 = item_off[z], it1 = item_off[z + 1];
  float s = 0.f;
  int it = it0;
  for (; it + 4 <= it1; it += 4) {
    const float a = spart[it * per + slot], b = spart[(it + 1) * per + slot];
    const float c = spart[(it + 2) * per + slot], d = spart[(it + 3) * per + slot];
    s += a; s += b; s += c; s += d;
  }
  for (; it < it1; it++) s += spart[it * per + slot];
  stot[(long long)z * per + slot] = s;
}

int reduce_items_launch(const float* spart, const int* item_off, int E, int npad, int K, float* stot, cudaStream_t st) {
  const long long per = (long long)npad * K;
  dim3 grid((unsigned)((per + 255) / 256), E);
  dw_reduce_items<<<grid, 256, 0, st>>>(spart, item_off, npad, K, stot);
  return 1;
}

size_t bucket_chunks(int64_t N) { return (size_t)((N + kChunk - 1) / kChunk); }

}  // namespace symcon

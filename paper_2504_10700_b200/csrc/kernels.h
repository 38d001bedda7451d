// Launch wrappers of the statically compiled (nvcc) kernels of libsymcon.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace symcon {

struct BucketArgs {
  const int* node_elem;
  int N, E, tile_nodes, tiles_per_item;
  int* hist;      // [nchunks][E+1]
  int* off;       // [nchunks][E+1]
  int* seg_off;   // [E+2]
  int* perm;      // [N]
  int4* tiles;    // [max_tiles]
  int* n_tiles;
  int4* items;    // [max_items]
  int* n_items;
  int* item_off;  // [E+2]
  int* tile_off;  // [E+1]
  int* tile_perm; // [max_tiles][tile_nodes], -1 padded
  int64_t max_tiles;
  int* chunk_bad;  // [nchunks] first out-of-range node of each chunk
  unsigned long long* err;
  int* zero_buf;   // zeroed by bk_scan (dW_r per-(element, channel block) item counters), may be NULL
  int zero_n;
  int fused;       // one cooperative kernel (bk_fused) instead of bk_hist + bk_scan + bk_scatter
};

int bucket_launch(const BucketArgs& a, cudaStream_t st);   // returns launches issued
int fill_nan_launch(const int* perm, const int* seg_off, int E, float* out, long long row, cudaStream_t st);
size_t bucket_chunks(int64_t N);
// stot[z][j][k] = sum over items it of element z (item order) of spart[it][j][k]
int reduce_items_launch(const float* spart, const int* item_off, int E, int npad, int K, float* stot, cudaStream_t st,
                        int parts_per_item = 1);   // parts_per_item -1: one part per item, single-item elements already in stot

// dW all-reduce over peer memory (peer.cu)
struct PeerArgs {
  const float* buf[8];   // each rank's symmetric dW buffer (peer pointers)
  unsigned* pad[8];      // each rank's signal pad (uint32 flags, slot r written by rank r)
  float* out[8];         // output of rank r (only out[rank] is used unless emulating)
};
// algo 1 one-shot, 2 two-shot (reduce-scatter + all-gather); spin_limit = barrier polls before
// the hard timeout (err = 1, NaN output); rank < 0 emulates all ranks on this device in one
// cooperative launch (blocks per rank x world). Returns launches issued, -1 on launch failure.
int peer_allreduce_launch(const PeerArgs& a, int world, int rank, long long n, unsigned epoch, unsigned* epoch_dev,
                          int algo, long long spin_limit, int* err, int blocks, cudaStream_t st);

// channelwise TP (tp_static.cu)
struct TPCsrArgs {
  const int* sender;
  const int* receiver;
  int N, E;
  unsigned long long* err;  // first bad edge (~0 = none)
  int* recv_off;            // [N+1]
  int* send_cnt;            // [N]      (sender CSR; all NULL to skip)
  int* send_off;            // [N+1]
  int* send_cur;            // [N]
  int* send_perm;           // [E]
  int* send_pos;            // [E] position of edge e in the sender CSR (inverse of send_perm)
  int skip_recv;            // 1: the check and recv_off are already in the workspace (graph reuse)
};
int tp_csr_launch(const TPCsrArgs& a, cudaStream_t st);
// dst[i] += src[i] for i < n (dst, src 16-byte aligned)
int add_inplace_launch(float* dst, const float* src, long long n, cudaStream_t st);
int tp_dh_reduce_launch(const float* dhe, const int* off, const int* perm, int N, int K, int nh, float* dh,
                        cudaStream_t st);

}  // namespace symcon

// Internal structures of libsymcon (product side; shares nothing with oracle/).
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/symcon.h"

namespace symcon {

void set_error(const std::string& msg);

// ---- cg.cpp: pairwise real coupling (ladder-operator construction)
// returns [(2L+1)][(2l1+1)][(2l2+1)] row-major; zeros if the triangle rule fails.
std::vector<double> real_coupling(int l1, int l2, int L);

// ---- builder.cpp
struct PathDesc {
  int L, nu, eta, col;
  std::array<int, 4> ls{{-1, -1, -1, -1}};
  std::array<int, 3> mids{{-1, -1, -1}};
};

struct SymRow {                 // one (L, M, monomial) row of the symmetrised table
  int L, M;                     // output irrep and component (M in [-L, L])
  int out;                      // per-channel output slot: off_L + M + L
  std::array<int, 4> mono;      // a <= b <= c <= d, padded with -1
  int deg;
  std::vector<std::pair<int, double>> cols;  // (path column, U~ value)
};

struct Tables {
  int lmax_in, corr, n_lm, E, K;
  std::vector<int> out_L, out_off;   // out_off[i] = sum_{j<i} (2 out_L[j] + 1)
  int out_per_ch;
  std::vector<PathDesc> paths;
  int64_t n_raw_terms = 0;
  std::vector<SymRow> rows;          // in codegen order (j index)
  int64_t n_sym_terms = 0;
  int n_monomials = 0;
  bool f64 = false;                  // fp64 plan
  bool simple = false;               // plain scalar kernels of codegen_simple.cpp (fp64, or correlation 4)
};

bool build_tables(int lmax_in, int corr, const std::vector<int>& out_L, int E, int K, Tables& t);

// ---- codegen.cpp
struct KernelConfig {
  int warps_per_cta = 8;     // dW kernel: channels per CTA (one warp per channel)
  int tile_sched = 0;        // fwd / dA: 0 strided items, 1 k-major contiguous ranges (coefficient reuse)
  int tile_warps = 1;        // fwd / dA persistent kernels: warps (channels) per CTA
  bool coef_tma = false;     // stage coefficients with cp.async.bulk + mbarrier (else per-lane cp.async)
  int tile_min_blocks = 1;   // __launch_bounds__ min blocks for fwd / dA (caps registers)
  int coef_batch = 0;        // >0: coefficient LDS in double-buffered batches of this many quads
  int coef_lookahead = 6;    // coefficient quads loaded ahead of first use
  int coef_mode = 0;         // coefficient staging: 0 per-lane cp.async, 2 registers (LDG.128) + STS
  bool coef_volatile = true; // issue coefficient LDS with volatile asm at the lookahead position
  bool coef_unroll = false;  // unroll the per-lane cp.async loop of the coefficient staging
  int tile_nodes = 64;       // nodes per tile (= 64 * node_pairs_per_lane; set by the plan)
  int node_pairs_per_lane = 1;  // fwd / dA: node pairs per lane (1 or 2)
  int acc_split = 1;         // fwd: independent partial accumulators per output (breaks FFMA2 chains)
  bool a_prefetch = true;    // fwd / dA: prefetch the next item's A / dB rows into registers
  int dw_tiles_per_item = 4; // tiles per dW work item
  int dw_tiles_per_butterfly = 2;  // tiles whose products are summed before one cross-lane reduction
  int dw_min_blocks = 2;           // __launch_bounds__ min blocks of the dW kernel
  int dw_rows_per_group = 0;       // transposed dW: rows j per warp (register accumulators); 0 = auto
  int dw_groups_per_cta = 0;       // transposed dW: warps per CTA; 0 = auto
  int bwd2_min_blocks = 10;        // double backward tile kernel: __launch_bounds__ min blocks (caps registers)
  int da_reserve_sms = 0;          // dA persistent grid leaves this many SMs free (for NCCL kernels at N > 1)
  int da_ctas_per_sm = 0;          // dA persistent grid: CTAs per SM (0 = occupancy maximum); fewer leave
                                   // room for concurrent dW CTAs on the same SMs
  int dw2_rows_per_group = 0;      // double-backward W_bar kernel (same layout): rows per warp; 0 = auto
  int dw2_groups_per_cta = 0;      // double-backward W_bar kernel: warps per CTA; 0 = auto
  int da_group = 0;                // dA: emit each prefix group's g first, then its D_c updates (operand reuse)
  int gamma = -1;                  // fwd (bit 1) / dA (bit 2) with lane = channel and register-resident
                                   // coefficients (few folded rows); -1 auto (dA only, rows <= 128)
  int dw_qform = -1;               // transposed dW: q = dB_o p_ab products shared by the prefix's rows; -1 auto
  int dw_np_unroll = 1;            // transposed dW: unroll of the node-pair loop (software pipelining)
  int dw_batch = 1;                // transposed dW: rows whose products are emitted before their FMAs
  int dw_block_nodes = 8;          // transposed dW: nodes per smem stage
  int unfold_channels = 8;   // channels per unfold CTA
  int fwd_r = -1;            // forward as symcon_fwd_r (lane = channel, warp = output slot, Horner); -1 auto
  int fwd_r_block = 16;       // fwd_r: nodes per shared-memory block (even, divides 64)
  int fwd_r_minb = 3;        // fwd_r: __launch_bounds__ min blocks (0 = none; 3 caps MP-medium at 170 registers)
  int fwd_r_ctas_per_sm = 0; // fwd_r: persistent CTAs per SM (0 = occupancy maximum)
  int dw_r = -1;             // dW as symcon_bwd_dW_r (lane = channel, warp = output slot, q-form); -1 auto
  int dw_r_block = 8;        // dw_r: nodes per shared-memory block
  int dw_r_minb = 0;         // dw_r: __launch_bounds__ min blocks
  int dw_r_unroll = 1;       // dw_r: node-loop unroll
  int fwd_r_nst = 2;         // fwd_r: TMA ring stages
  int dw_r_nst = 2;          // dw_r: TMA ring stages
  int dw_r_split = 1;        // dw_r: warps per output slot (each takes a balanced range of first indices a)
  int bucket_fused = 0;      // element bucketing as one cooperative kernel (bk_fused)
  int fwd_r_tr = 0;          // fwd_r: interleave the block's node pairs once in shared memory (no per-warp pairing)
  int unfold_reduce = 0;     // the unfold kernel sums the element's dW item partials itself (no dw_reduce_items)
  int fwd_r_npw = 1;         // fwd_r: node pairs per warp iteration (1 or 2)
  int r_rotate = 1;          // fwd_r / dW_r: rotate the warp -> output slot map by CTA
  int fold_split = 4;        // W-fold: CTAs per (element, 32-channel block) (grid.z)
  int dw_r_fuse = 0;         // dw_r: the last CTA of each (element, channel block) reduces + unfolds in-kernel
  int da_s = -1;             // dA as symcon_bwd_dA_s (one node per lane, scalar FP32); -1 auto
  int da_s_warps = 4;        // da_s: warps (channels) per CTA
  int da_s_minb = 0;         // da_s: __launch_bounds__ min blocks
  int simple_warps = 4;      // simple plans (fp64 / corr 4): warps per fwd / dA CTA (coefficient rows in dynamic smem)
  int simple_unfold_split = 1;  // simple plans: column split of the unfold grid (grid.z)
  int simple_rpg = 0;        // simple plans: dW rows per warp (register accumulators); 0 auto (fp32 128, fp64 96)
  int fwd_r_split = 1;       // fwd_r: 2 = two warps per output slot (each half of the first indices), partial B summed in smem
  int fwd_r_prod_light = 1;  // fwd_r: the TMA producer is the warp of the lightest slot (else the CTA's warp 0)
  int dw_r_balance = 0;      // dW_r: warps take (slot, first index) units balanced by op count instead of whole slots
  int dw_r_prod_light = 1;   // dW_r: the TMA producer is the warp with the lightest row group (else row group 0)
  int dw_r_unfold_single = 1;   // dW_r CTAs of single-item elements unfold dW themselves (skipped by reduce / unfold)
  int gamma_split = 0;       // gamma dA: warps per tile (grid.z) splitting its nodes; 0 auto (fill the GPU's warp slots)
  int dw_r_wps = 0;          // dW_r: warps per output slot (each its own partial over every wps-th node of a stage); 0 auto
  int dw_r_groups = 0;       // dW_r: CTAs (grid.z) per (item, channel block), each a subset of the row groups; 0 auto
  int fwd_r_groups = 0;      // fwd_r: CTAs per node block, each serving 1/groups of the output slots; 0 auto
  int fwd_r_wps = 0;         // fwd_r: warps per output slot, each taking every wps-th node pair of a stage; 0 auto
  int fwd_r_chains = 2;      // fwd_r: 2 (measured -2% fwd time) splits the Horner T / B accumulation chains into even / odd halves
  int fold_fork = 1;         // run the W-fold on an auxiliary stream concurrently with the bucketing
  int dw_items_adapt = 1;    // lower the tiles per dW item for small N (dW_r plans; api.cpp tiles_per_item)
};
std::string generate_source(const Tables& t, const KernelConfig& kc);
// codegen_simple.cpp: plain scalar kernels of any degree (prefix-trie forward, reverse-mode dA), fp32 or fp64
std::string generate_source_simple(const Tables& t, const KernelConfig& kc);

// Horner program of one output slot (symcon_fwd_r)
struct HornerB { int b, row_ab; std::vector<std::pair<int, int>> cs; };   // (c, row j) of degree-3 rows
struct HornerA { int a, row_a; std::vector<HornerB> bs; int slot = -1; };   // slot: set when a warp mixes slots
struct HornerSlot { int slot; std::vector<HornerA> as; std::vector<int> rows; int half = 0; };  // rows: register order
std::vector<HornerSlot> horner_slots(const Tables& t);
// fwd_r warps: the slots, or (fwd_r_split = 2) each slot's first indices split in two op-balanced halves
// (slot-major: [s0 h0, s0 h1, s1 h0, ...]); the coefficient table coef_r is laid out per entry
std::vector<HornerSlot> horner_vslots(const Tables& t, int split);
int64_t horner_ops(const Tables& t);
std::string generate_fwd_r(const Tables& t, const KernelConfig& kc);
std::string generate_dw_r(const Tables& t, const KernelConfig& kc);
std::string generate_da_s(const Tables& t, const KernelConfig& kc);
// apply "key=value,..." overrides (env SYMCON_KCONFIG) to a KernelConfig; returns false on bad keys
bool parse_kernel_config(const char* spec, KernelConfig& kc);

// ---- api.cpp helpers shared with tp.cpp
bool compile_cubin(const std::string& src, std::vector<char>& cubin);  // NVRTC sm_100a + disk cache

// ---- pack.cpp
int64_t pack_balanced(const int64_t* sizes, int64_t n, int64_t C, int G,
                      std::vector<std::vector<int64_t>>& bins);

}  // namespace symcon

/* symcon.h — C ABI of libsymcon.so: MACE's symmetric tensor contraction on B200 (sm_100a).
 *
 * Operation (arXiv 2504.10700, Alg. 3; Eq. (2)):
 *   for node i, channel k, output irrep L in out_L, component M:
 *     B[i,k,(L,M)] = sum_{nu=1..correlation} sum_eta W[z_i,(L,nu,eta),k]
 *                    * sum_{lm_1..lm_nu} U^{LM}_{nu,eta,lm_1..lm_nu} * prod_j A[i,k,lm_j]
 *   U is the generalized real Clebsch-Gordan coefficient C^{LM}_{lm},
 *   read as a left-nested chain of pairwise real couplings (DESIGN.md §3 reading s4), with
 *   the CG selection rules of PAPER.md:696-697. W is per element ("depends on the atomic
 *   species z_i"). Backward: dA (forces are derivatives of the energy,
 *   PAPER.md:331) and dW.
 *
 * Layouts (all row-major, fp32 unless noted):
 *   A, dA     [N][K][(lmax_in+1)^2]            lm = l*l + l + m fastest
 *   B, dB     [N][sum_L K*(2L+1)]              per-L block [K][2L+1], blocks in out_L order
 *   W, dW     [E][P][K]                        P = symcon_info.n_paths; columns ordered by
 *                                              out_L, then nu, then eta (symcon_plan_path)
 *   node_elem int32 [N], values in [0, E)
 *
 * Ownership: the caller owns every device buffer (A, W, node_elem, B, dA, dB, dW and the
 * workspace); the library owns only the plan (host tables, device tables, loaded kernels),
 * freed by symcon_destroy. All device pointers live on the plan's device. Calls are
 * asynchronous on the given stream; no host synchronisation except where stated.
 *
 * Errors: invalid arguments are reported synchronously (before any launch) as
 * SYMCON_EINVAL / SYMCON_EUNSUPPORTED; CUDA launch failures as SYMCON_ECUDA. An
 * out-of-range node_elem value is detected on the device: that node's outputs (B row, dA
 * row) are set to NaN, it contributes nothing to dW, and the first offending node index is
 * recorded in the workspace; symcon_check_device_error (synchronising) returns
 * SYMCON_EELEMENT for it ("species index without weights -> validation error").
 *
 * Determinism: no floating-point atomics; dW is reduced in a fixed order, so all outputs
 * are bitwise reproducible for a given (plan, N, node_elem, inputs, device).
 * Thread-safety: a plan is immutable after symcon_build_tables; concurrent calls on
 * different streams are allowed when each call has its own workspace.
 */
#ifndef SYMCON_H
#define SYMCON_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SYMCON_OK = 0,
  SYMCON_EINVAL = 1,       /* bad argument (null pointer, size, alignment, range) */
  SYMCON_EUNSUPPORTED = 2, /* valid but not supported (e.g. correlation > 4) */
  SYMCON_ECUDA = 3,        /* CUDA / NVRTC failure */
  SYMCON_ENOMEM = 4,       /* host allocation or workspace too small */
  SYMCON_EELEMENT = 5,     /* node_elem value outside [0, E) found on the device */
  SYMCON_ETIMEOUT = 6      /* peer all-reduce: a rank did not reach the barrier (symcon_peer_check) */
} symcon_status;

typedef struct symcon_plan symcon_plan; /* opaque */

typedef struct {
  int32_t lmax_in, correlation, n_out, num_elements, channels;
  int32_t out_L[4];
  int32_t eta[4][4];     /* eta[out index][nu-1]: number of paths */
  int64_t n_paths;       /* P: W middle dimension */
  int64_t weight_numel;  /* E * P * K */
  int64_t in_dim;        /* K * (lmax_in+1)^2  per node */
  int64_t out_dim;       /* K * sum_L (2L+1)   per node */
  int64_t n_raw_terms;   /* raw ordered-tuple U nonzeros, all paths */
  int64_t n_sym_terms;   /* (L,M,monomial,path) nonzeros after symmetrisation */
  int64_t n_fold;        /* (L,M,monomial) rows: folded coefficients per (element, channel) */
  int64_t n_monomials;   /* distinct monomials of A used */
  int32_t device;        /* -1: host-only plan (tables, no kernels) */
  int32_t reserved;      /* the plan's dtype (SYMCON_F32 / SYMCON_F64) */
} symcon_info;

/* Arithmetic type of a plan (symcon_build_tables_ex). */
#define SYMCON_F32 0
#define SYMCON_F64 1

/* Build the U tables for (lmax_in, correlation, out_L[0..n_out)) and, if device >= 0,
 * generate, compile (NVRTC, sm_100a; cached on disk) and load the kernels for that device.
 *   lmax_in in [0,3]; correlation in [1,4]; out_L strictly increasing, each in [0,3],
 *   n_out in [1,4]; num_elements >= 1; channels >= 1.
 *   Correlation 4 ("all possible combinations" at nu = 4; reading s4b: every
 *   nu = 4 intermediate has natural parity and L_j < 12) builds the plain scalar kernels of any
 *   degree (fp32 or fp64); the double backward (symcon_backward2*) is correlation <= 3 only.
 *   device = -1 builds host tables only (for inspection; compute calls return EINVAL).
 * On success *plan is owned by the caller and must be freed with symcon_destroy. */
symcon_status symcon_build_tables(int lmax_in, int correlation, const int* out_L, int n_out,
                                  int num_elements, int channels, int device, symcon_plan** plan);

/* The same with the arithmetic type: SYMCON_F32 (the fp32 kernels; every call below) or SYMCON_F64
 * (the paper's Float64 runs): every float array of the
 * forward / backward is double and the calls are symcon_forward_f64 / symcon_backward_f64 (same
 * layouts, workspace from symcon_workspace_bytes of the fp64 plan). The double backward and the
 * peer all-reduce are fp32 only. symcon_info.reserved reports the plan's dtype. */
symcon_status symcon_build_tables_ex(int lmax_in, int correlation, const int* out_L, int n_out,
                                     int num_elements, int channels, int device, int32_t dtype,
                                     symcon_plan** plan);

symcon_status symcon_plan_info(const symcon_plan* plan, symcon_info* info);

/* Describe W column `col` in [0, P): its output L, order nu, index eta, the coupled
 * irreps ls[0..nu) and the intermediates mids[0..nu-1) (mids[nu-2] == L for nu >= 2). */
symcon_status symcon_plan_path(const symcon_plan* plan, int64_t col, int32_t* L, int32_t* nu,
                               int32_t* eta, int32_t* ls, int32_t* mids);

/* Copy the symmetrised table (host): rows (L, M, monomial a<=b<=c padded with -1, path
 * column, value). Pass NULL arrays to query the count into *n. Used by table-parity tests.
 * A correlation-4 plan returns EUNSUPPORTED when mono3 is requested (use symcon_plan_sym_table4). */
symcon_status symcon_plan_sym_table(const symcon_plan* plan, int64_t* n, int32_t* L, int32_t* M,
                                    int32_t* mono3, int32_t* col, double* value);

/* The same with 4 monomial indices per row (a<=b<=c<=d padded with -1): mono4[4 * n]. */
symcon_status symcon_plan_sym_table4(const symcon_plan* plan, int64_t* n, int32_t* L, int32_t* M,
                                     int32_t* mono4, int32_t* col, double* value);

/* Copy the pairwise real coupling C^L_{l1 l2}[M][m1][m2] (host) into out
 * [(2L+1)(2l1+1)(2l2+1)] (zeros if the triangle rule fails). l1,l2 <= 3, L <= 6. */
symcon_status symcon_real_cg(int l1, int l2, int L, double* out);

/* Workspace bytes needed by forward/backward for num_nodes nodes (16-byte aligned). */
size_t symcon_workspace_bytes(const symcon_plan* plan, int64_t num_nodes);

/* Forward: B (overwritten) from A, W, node_elem. N = 0 is a no-op. A and B 16-byte
 * aligned. ws must hold symcon_workspace_bytes(plan, num_nodes) bytes. */
symcon_status symcon_forward(const symcon_plan* plan, int64_t num_nodes, const float* A,
                             const float* W, const int32_t* node_elem, float* B, void* ws,
                             size_t ws_bytes, void* stream /* cudaStream_t */);

/* Backward: dA (overwritten, may be NULL to skip) and dW (overwritten, may be NULL to skip)
 * from A, W, node_elem and the cotangent dB. Elements without nodes get dW = 0. */
symcon_status symcon_backward(const symcon_plan* plan, int64_t num_nodes, const float* A,
                              const float* W, const int32_t* node_elem, const float* dB, float* dA,
                              float* dW, void* ws, size_t ws_bytes, void* stream /* cudaStream_t */);

/* fp64 plans (SYMCON_F64): forward and backward on double arrays, same semantics and layouts as
 * symcon_forward / symcon_backward_ex (flags: SYMCON_REUSE_*). An fp32 plan returns EINVAL. */
symcon_status symcon_forward_f64(const symcon_plan* plan, int64_t num_nodes, const double* A,
                                 const double* W, const int32_t* node_elem, double* B, void* ws,
                                 size_t ws_bytes, void* stream /* cudaStream_t */);
symcon_status symcon_backward_f64(const symcon_plan* plan, int64_t num_nodes, const double* A,
                                  const double* W, const int32_t* node_elem, const double* dB, double* dA,
                                  double* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                  void* stream /* cudaStream_t */);

/* Reuse hints for symcon_backward_ex (a training step calls forward then backward with the
 * same node_elem and W on the same workspace):
 *   SYMCON_REUSE_BUCKETS  skip the element bucketing if the last call on `ws` used the same
 *                         num_nodes and node_elem pointer (the caller promises unchanged contents);
 *   SYMCON_REUSE_FOLD     additionally skip the W-fold if that call also used the same W pointer.
 * Hints never change results: when the recorded pointers differ the work is redone. */
#define SYMCON_REUSE_BUCKETS 1u
#define SYMCON_REUSE_FOLD 2u
symcon_status symcon_backward_ex(const symcon_plan* plan, int64_t num_nodes, const float* A,
                                 const float* W, const int32_t* node_elem, const float* dB, float* dA,
                                 float* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                 void* stream /* cudaStream_t */);

/* Double backward: training on forces differentiates the backward
 * itself (forces F = -dE/dr enter the loss; MACE trains on energies and
 * forces). Given the cotangent uA [N][K][n_lm] of dA, returns the derivatives of
 * <uA, dA(A, W, dB)>:
 *   dB_bar [N][out_dim]   = sum_paths W U (grad_A monomial . uA)      (the JVP of the forward)
 *   A_bar  [N][K][n_lm]   = sum_M dB_M sum_paths W U Hess_A(monomial) uA
 *   W_bar  [E][P][K]      = sum_{i of element z} sum_M dB_M U (grad_A monomial . uA)
 * (raw-tuple definitions: oracle/contraction.py backward2). Each output is overwritten and may
 * be NULL to skip it; W_bar of elements without nodes is 0. A, dB, uA, dB_bar and A_bar must be
 * 16-byte aligned; same shapes, workspace, flags (SYMCON_REUSE_*) and error behaviour as
 * symcon_backward_ex. The cotangent of dW (uW) needs no kernel of its own: its terms are
 * symcon_forward (dB_bar += forward(A, uW)) and symcon_backward dA (A_bar += dA(A, uW, dB)). */
symcon_status symcon_backward2(const symcon_plan* plan, int64_t num_nodes, const float* A,
                               const float* W, const int32_t* node_elem, const float* dB,
                               const float* uA, float* dB_bar, float* A_bar, float* W_bar, void* ws,
                               size_t ws_bytes, uint32_t flags, void* stream /* cudaStream_t */);
/* The full double backward of (A, W, dB) -> (dA, dW) with cotangents (uA, uW): the uA terms as in
 * symcon_backward2 plus the uW terms, computed in libsymcon (no caller arithmetic):
 *   dB_bar += forward(A, uW)   and   A_bar += dA(A, uW, dB)   (W_bar gets no uW term: dW is linear in dB
 *   and independent of W). uA or uW may be NULL (not both); the outputs are overwritten. */
symcon_status symcon_backward2_ex(const symcon_plan* plan, int64_t num_nodes, const float* A,
                                  const float* W, const int32_t* node_elem, const float* dB,
                                  const float* uA, const float* uW, float* dB_bar, float* A_bar, float* W_bar,
                                  void* ws, size_t ws_bytes, uint32_t flags, void* stream /* cudaStream_t */);

/* Synchronises `stream`; returns SYMCON_EELEMENT and *first_bad_node if the last forward /
 * backward that used `ws` saw an out-of-range node_elem, SYMCON_ECUDA on a CUDA error. */
symcon_status symcon_check_device_error(const symcon_plan* plan, void* ws, void* stream,
                                        int64_t* first_bad_node);

/* Kernel launches the last forward/backward on this plan issued (for bench accounting). */
int32_t symcon_last_launch_count(const symcon_plan* plan);

/* Optional launch timer for benchmarking: when enabled, every launch group (bucket, fold,
 * fwd, bwd_dA, bwd_dW, unfold, bwd2, bwd2_dW) is bracketed by CUDA events on its stream.
 * symcon_profile_read synchronises those events and returns up to SYMCON_PROFILE_MAX entries of
 * (kernel name, launches, total milliseconds); names point to static strings. */
#define SYMCON_PROFILE_MAX 12
symcon_status symcon_profile_enable(const symcon_plan* plan, int on);
symcon_status symcon_profile_reset(const symcon_plan* plan);
int32_t symcon_profile_read(const symcon_plan* plan, const char** names, int64_t* counts, double* total_ms);

/* Build-host helpers (no device needed): NVRTC-compile a configuration's kernels into the
 * cubin cache and report its path; copy a plan's generated CUDA source (NULL buf: size). */
symcon_status symcon_precompile(int lmax_in, int correlation, const int* out_L, int n_out, char* path,
                                size_t path_len);
symcon_status symcon_precompile_ex(int lmax_in, int correlation, const int* out_L, int n_out, int32_t dtype,
                                   char* path, size_t path_len);
size_t symcon_plan_source(const symcon_plan* plan, char* buf, size_t len);

void symcon_destroy(symcon_plan* plan);
const char* symcon_status_string(symcon_status s);
/* Human-readable detail of the last error in this thread (never NULL). */
const char* symcon_last_error(void);

/* ---- host partitioner (Alg. 1 Create-Balanced-Batches) -------------
 * sizes[n] >= 0 (graph vertex counts), capacity C, workers G >= 1. Produces bins in
 * creation order: bin b holds graph_ids[bin_offsets[b] .. bin_offsets[b+1]).
 * Bin b runs on rank b % G at step b / G (reading s18). Deterministic.
 * Any size > C -> SYMCON_EINVAL. If max_bins is too small -> SYMCON_ENOMEM with *n_bins
 * set to the required count. bin_offsets needs max_bins+1 entries, graph_ids n entries. */
symcon_status symcon_pack_balanced(const int64_t* sizes, int64_t n, int64_t capacity,
                                   int32_t workers, int64_t* bin_offsets, int64_t* graph_ids,
                                   int64_t max_bins, int64_t* n_bins);

/* ---- dW all-reduce over NVLink peer memory ("all-reduce") ------
 * The data-parallel step's one exchange: dW = sum over ranks of each rank's partial.
 * bufs[r] (r < world <= 8): device pointer, valid on this GPU (peer mapping), of rank r's
 * n-float partial, 16-byte aligned; pads[r]: rank r's signal pad (>= 2*world + 1 uint32 slots,
 * zero-initialised, peer mapped; slot 2*world is this rank's private grid counter).
 * One kernel per call (plus, in the _dev form, a one-thread epoch bump):
 *   algo 1, one-shot: a cross-GPU barrier (this rank writes `epoch` to slot `rank` of every pad,
 *     then waits until slots [0, world) of its own pad reach `epoch`; epochs must increase by
 *     call), then out[i] = sum_{r = 0..world-1} bufs[r][i] in rank order.
 *   algo 2, two-shot: the same barrier; rank r sums slice r of all partials (rank order) in place
 *     into slice r of bufs[r]; a second barrier on slots [world, 2 world); out gathers slice q
 *     from bufs[q]. NVLink reads per rank: 2 (world-1)/world x n floats instead of (world-1) x n.
 *   algo 0: auto (two-shot for world >= 8; one-shot measured faster at 2 and 4 GPUs).
 * Every rank ends with bitwise the same out (each element summed once, in rank order).
 * The caller must not overwrite bufs[rank] until every rank's call has completed (alternate two
 * buffers per step); with algo 2, bufs[rank] is modified. out must not alias any bufs[r].
 * Error: a barrier that does not complete within spin_limit polls of ~200 ns (0 = default 2^26,
 * tens of seconds) is a hard error: *err (device int32, may be NULL) is set to 1 and `out` is
 * filled with NaN, never with partial sums; symcon_peer_check reports it as SYMCON_ETIMEOUT. */
symcon_status symcon_peer_allreduce_ex(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                       int64_t n, uint32_t epoch, uint32_t* epoch_counter, int32_t algo,
                                       int64_t spin_limit, float* out, int32_t* err, void* stream);
/* epoch_counter (nullable): if non-NULL the epoch is read on the device as *epoch_counter + 1 (a
 * uint32 in device memory, zero-initialised, one per reducer) and the counter is incremented by a
 * one-thread kernel right after, so a call captured in a CUDA graph can be replayed; `epoch` is
 * then ignored. */
/* Legacy forms: one-shot with a host epoch / with a device epoch counter, default spin limit. */
symcon_status symcon_peer_allreduce(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                    int64_t n, uint32_t epoch, float* out, int32_t* err, void* stream);
symcon_status symcon_peer_allreduce_dev(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                        int64_t n, uint32_t* epoch_counter, float* out, int32_t* err, void* stream);
/* Diagnostic form for one GPU: the all-reduce of `world` ranks whose buffers (bufs, pads, outs; all
 * on this device) are all here, run as ONE cooperative launch in which each rank's blocks execute
 * the same kernel code as symcon_peer_allreduce_ex (rank = blockIdx.y), so the barrier protocol,
 * the two-shot slices and the rank-order sums are exercised without several GPUs (ranks that wait
 * on one another must not be separate launches on one GPU). algo 1 or 2. */
symcon_status symcon_peer_allreduce_emulate(const float* const* bufs, uint32_t* const* pads, float* const* outs,
                                            int32_t world, int64_t n, uint32_t epoch, int32_t algo, int64_t spin_limit,
                                            int32_t* err, void* stream);
/* Synchronises `stream` and reads *err: SYMCON_ETIMEOUT if a barrier of an earlier call timed out. */
symcon_status symcon_peer_check(const int32_t* err, void* stream);

/* ---- channelwise tensor product + edge->node sum ----------------
 * Alg. 2 of the paper, the message construction that feeds the contraction,
 * with the neighbour sum of Eq. (1):
 *
 *   A[i,k,l3 m3] = sum_{e: receiver[e] = i} sum_{paths p = (l1,l2,l3)} R[e,k,p]
 *                  sum_{m1,m2} C^{l3 m3}_{l1 m1, l2 m2} Y[e, l1 m1] h[sender[e], k, l2 m2]
 *
 * C is the real coupling of symcon_real_cg. Paths: every (l1 <= lmax_y, l2 in hidden_l,
 * l3 <= lmax_out) with |l1-l2| <= l3 <= l1+l2 and l1+l2+l3 even, ordered by (l1, l2, l3)
 * (symcon_tp_path). Layouts (fp32, row-major, 16-byte aligned):
 *   Y [E][(lmax_y+1)^2]  (lm = l^2+l+m)       h  [N][n_h][K] (hidden blocks in hidden_l order,
 *                                                 channel fastest)
 *   R [E][n_paths][K] (channel fastest, e3nn's per-path weight blocks)
 *                                              A  [N][K][(lmax_out+1)^2] (the contraction's A)
 *   sender, receiver: int32 [E]; receiver must be non-decreasing (edges sorted by receiver);
 *   a violation or an index outside [0, N) is reported by symcon_tp_check_device_error
 *   (SYMCON_EINVAL) and the outputs are unspecified. Nodes without incoming edges get A = 0.
 * The backward returns the derivatives of <dA, A>: dY [E][n_y], dh [N][n_h][K] and
 * dR [E][n_paths][K] (each overwritten; any may be NULL). Deterministic: fixed summation
 * order, no floating-point atomics. */
typedef struct symcon_tp_plan symcon_tp_plan; /* opaque */

/* hidden_l: n_hidden strictly increasing irrep orders in [0,3]; lmax_y, lmax_out in [0,3];
 * channels K >= 1. device < 0: host-only plan (tables and source, no kernels). */
symcon_status symcon_tp_build(int lmax_y, const int* hidden_l, int n_hidden, int lmax_out, int channels,
                              int device, symcon_tp_plan** plan);
/* Build-host helper (no device needed): NVRTC-compile a TP configuration's kernels (they depend
 * on K) into the cubin cache. */
symcon_status symcon_tp_precompile(int lmax_y, const int* hidden_l, int n_hidden, int lmax_out, int channels);
/* n_paths, n_y = (lmax_y+1)^2, n_h, n_out = (lmax_out+1)^2 */
symcon_status symcon_tp_info(const symcon_tp_plan* plan, int32_t* n_paths, int32_t* n_y, int32_t* n_h,
                             int32_t* n_out);
symcon_status symcon_tp_path(const symcon_tp_plan* plan, int32_t p, int32_t* l1, int32_t* l2, int32_t* l3);
size_t symcon_tp_workspace_bytes(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges);
symcon_status symcon_tp_forward(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                const float* Y, const float* h, const float* R, const int32_t* sender,
                                const int32_t* receiver, float* A, void* ws, size_t ws_bytes,
                                void* stream /* cudaStream_t */);
symcon_status symcon_tp_backward(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                 const float* Y, const float* h, const float* R, const int32_t* sender,
                                 const int32_t* receiver, const float* dA, float* dY, float* dh, float* dR,
                                 void* ws, size_t ws_bytes, void* stream /* cudaStream_t */);
/* The same with flags: SYMCON_TP_REUSE_GRAPH keeps the graph structure (the receiver-offset check and
 * CSR, and the sender CSR of the backward) that the last TP call on `ws` built for the same sender /
 * receiver pointers, N and E; the caller guarantees the index arrays are unchanged since that call
 * (e.g. the backward of a step after its forward). Otherwise (or on any mismatch) it is rebuilt. */
#define SYMCON_TP_REUSE_GRAPH 4u
/* Forward flag: also build the backward's sender CSR into `ws`, on an internal stream concurrently with
 * the forward kernel (joined before the call's work on `stream` completes); a following backward with
 * SYMCON_TP_REUSE_GRAPH then builds nothing. */
#define SYMCON_TP_PREP_BACKWARD 8u
symcon_status symcon_tp_forward_ex(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                   const float* Y, const float* h, const float* R, const int32_t* sender,
                                   const int32_t* receiver, float* A, void* ws, size_t ws_bytes, uint32_t flags,
                                   void* stream);
symcon_status symcon_tp_backward_ex(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                    const float* Y, const float* h, const float* R, const int32_t* sender,
                                    const int32_t* receiver, const float* dA, float* dY, float* dh, float* dR,
                                    void* ws, size_t ws_bytes, uint32_t flags, void* stream);
/* Double backward of the TP (the derivatives of <(uY, uh, uR), (dY, dh, dR)(Y, h, R, dA)> and of <uA_bar...>:
 * the TP is linear in each of Y, h, R, so every term is a TP pass with one input replaced by its
 * cotangent, summed on the device (no caller arithmetic):
 *   dA_bar = TP(uY,h,R) + TP(Y,uh,R) + TP(Y,h,uR)
 *   Y_bar  = dY|(h:=uh) + dY|(R:=uR),  h_bar = dh|(R:=uR) + dh|(Y:=uY),  R_bar = dR|(h:=uh) + dR|(Y:=uY)
 * Outputs overwritten, any may be NULL. ws needs symcon_tp_workspace2_bytes (the TP workspace plus
 * one temporary of each output's size). */
size_t symcon_tp_workspace2_bytes(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges);
symcon_status symcon_tp_backward2(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                  const float* Y, const float* h, const float* R, const int32_t* sender,
                                  const int32_t* receiver, const float* dA, const float* uY, const float* uh,
                                  const float* uR, float* dA_bar, float* Y_bar, float* h_bar, float* R_bar,
                                  void* ws, size_t ws_bytes, void* stream /* cudaStream_t */);
/* The same with flags (SYMCON_TP_REUSE_GRAPH for the first of its six passes; the other five always
 * reuse the structure the first one built). */
symcon_status symcon_tp_backward2_ex(const symcon_tp_plan* plan, int64_t num_nodes, int64_t num_edges,
                                     const float* Y, const float* h, const float* R, const int32_t* sender,
                                     const int32_t* receiver, const float* dA, const float* uY, const float* uh,
                                     const float* uR, float* dA_bar, float* Y_bar, float* h_bar, float* R_bar,
                                     void* ws, size_t ws_bytes, uint32_t flags, void* stream);
/* Synchronises `stream`; SYMCON_EINVAL if the last TP call on `ws` saw unsorted receivers or an
 * out-of-range node index (*first_bad_edge = the first such edge), SYMCON_ECUDA on CUDA errors. */
symcon_status symcon_tp_check_device_error(const symcon_tp_plan* plan, void* ws, void* stream,
                                           int64_t* first_bad_edge);
int32_t symcon_tp_last_launch_count(const symcon_tp_plan* plan);
size_t symcon_tp_source(const symcon_tp_plan* plan, char* buf, size_t len);
void symcon_tp_destroy(symcon_tp_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* SYMCON_H */

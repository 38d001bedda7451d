// C ABI of libsymcon (include/symcon.h): plan construction, NVRTC kernel compilation with an
// on-disk cubin cache, workspace carving and the forward / backward launch sequences.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.h"

namespace symcon {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace symcon

using namespace symcon;

struct symcon_plan {
  Tables t;
  KernelConfig kc;
  int device = -1;
  int npad = 0;
  size_t unfold_smem = 0, tile_smem = 0, dw_smem = 0, dw2_smem = 0;
  int dw_gpc = 1, dw_nz = 1, dw2_gpc = 1, dw2_nz = 1;
  int grid_fwd = 0, grid_dA = 0, grid_bwd2 = 0, grid_fwd_r = 0;
  int rnq = 0;                 // fwd_r: coefficient quads per output slot
  int warp_slots_dA_g = 0;     // gamma dA: resident warps over the GPU (tile split heuristic)
  size_t fwd_r_smem = 0;
  size_t simple_smem = 0;                               // simple plans: dynamic smem of fwd / dA
  std::string source;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t k_fold = nullptr, k_fwd = nullptr, k_dA = nullptr, k_dW = nullptr, k_unfold = nullptr;
  cudaKernel_t k_bwd2 = nullptr, k_bwd2_dW = nullptr;
  cudaKernel_t k_fwd_g = nullptr, k_dA_g = nullptr;   // gamma variants (kc.gamma)
  cudaKernel_t k_fwd_r = nullptr;                      // output-slot warps, Horner (kc.fwd_r)
  cudaKernel_t k_dW_r = nullptr;                       // output-slot warps, q-form (kc.dw_r)
  cudaKernel_t k_dA_s = nullptr;                       // one node per lane, scalar (kc.da_s)
  cudaKernel_t k_reduce_s = nullptr;                   // simple plans (fp64 / corr 4): the dW item reduction
  size_t da_s_smem = 0;
  int grid_dA_s = 0;
  size_t dw_r_smem = 0;
  mutable std::atomic<int> last_launches{0};
  // the W-fold runs on this stream concurrently with the element bucketing (fork / join by events;
  // works under stream capture)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  mutable std::mutex fork_mu;
  // optional launch timer (symcon_profile_*): CUDA events around each launch group
  struct Rec { int kind; cudaEvent_t a, b; };
  mutable std::mutex prof_mu;
  mutable bool prof_on = false;
  mutable std::vector<Rec> recs;
  mutable std::vector<cudaEvent_t> event_pool;
  mutable double prof_ms[SYMCON_PROFILE_MAX] = {0};
  mutable int64_t prof_n[SYMCON_PROFILE_MAX] = {0};
  // per-workspace record of what the last call left in it (for the SYMCON_REUSE_* hints)
  struct WsState { int64_t N = -1; const void* ne = nullptr; const void* W = nullptr; };
  mutable std::mutex ws_mu;
  mutable std::map<const void*, WsState> ws_state;
};

static const char* kKindNames[] = {"symcon_bucket", "symcon_fold", "symcon_fwd", "symcon_bwd_dA", "symcon_bwd_dW",
                                   "symcon_unfold", "symcon_fill_nan", "symcon_bwd2", "symcon_bwd2_dW"};
enum { K_BUCKET = 0, K_FOLD, K_FWD, K_DA, K_DW, K_UNFOLD, K_NAN, K_BWD2, K_BWD2_DW, K_NKINDS };
static_assert(K_NKINDS <= SYMCON_PROFILE_MAX, "profile table");

namespace {
cudaEvent_t take_event(const symcon_plan* p) {
  if (!p->event_pool.empty()) { cudaEvent_t e = p->event_pool.back(); p->event_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void drain(const symcon_plan* p) {  // caller holds prof_mu
  for (auto& r : p->recs) {
    float ms = 0;
    if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      p->prof_ms[r.kind] += ms;
      p->prof_n[r.kind]++;
    }
    p->event_pool.push_back(r.a);
    p->event_pool.push_back(r.b);
  }
  p->recs.clear();
}
struct Timed {  // RAII: records start/stop events around a launch group when profiling is on
  const symcon_plan* p; int kind; cudaStream_t st; cudaEvent_t a = nullptr, b = nullptr;
  Timed(const symcon_plan* p_, int k, cudaStream_t s) : p(p_), kind(k), st(s) {
    if (!p->prof_on) return;
    std::lock_guard<std::mutex> g(p->prof_mu);
    if (p->recs.size() > 4096) drain(p);
    a = take_event(p); b = take_event(p);
    cudaEventRecord(a, st);
  }
  ~Timed() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> g(p->prof_mu);
    p->recs.push_back({kind, a, b});
  }
};
}  // namespace

namespace {

struct alignas(64) TmapA { unsigned long long d[16]; };   // CUtensorMap
static_assert(sizeof(TmapA) == sizeof(CUtensorMap), "tensor map size");
struct Params {  // must match SymconParams in codegen.cpp
  const float* A; const float* W; const int* node_elem; const float* dB;
  float* B; float* dA; float* dW;
  const int* perm; const int4* tiles; const int* n_tiles; const int4* items; const int* n_items;
  const int* item_off; const int* seg_off;
  float* coef; float* spart;
  int N, K, E, pad;
  float zero;
  const int* tile_perm;
  float* stot;
  const float* U;
  float* coef_r;
  int* dw_count;
  int accum;
  TmapA tmA;
};

// TMA descriptor of A viewed as [N*K rows][16 floats] (row = (node, channel)), box 32 rows x 16 floats
// (one node's 32-channel block, 2 KB), 64-byte swizzle (the R kernels read it conflict-free), zero fill
// past the end. The driver entry point is looked up once (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
symcon_status encode_a_map(TmapA& m, const float* A, int64_t N, int K, int n_lm) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  });
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return SYMCON_ECUDA; }
  const cuuint64_t dims[2] = {(cuuint64_t)n_lm, (cuuint64_t)N * (cuuint64_t)K};
  const cuuint64_t strides[1] = {(cuuint64_t)n_lm * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)n_lm, 32u};
  const cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(&m), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r)); return SYMCON_ECUDA; }
  return SYMCON_OK;
}

struct WsLayout {
  size_t hist, chunk_bad, off, seg_off, perm, tiles, n_tiles, items, n_items, item_off, err, coef, spart, tile_off, tile_perm, stot,
      coef_r, dw_count, coef2, coef_r2, total;
  int64_t max_tiles, max_items;
};

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

size_t esz(const symcon_plan* p) { return p->t.f64 ? sizeof(double) : sizeof(float); }

// threads of a symcon_fwd_r CTA: (slots x split halves) / slot groups x warps per entry
int fwd_r_threads(const symcon_plan* p) {
  return 32 * p->t.out_per_ch * p->kc.fwd_r_split / std::max(1, p->kc.fwd_r_groups) * std::max(1, p->kc.fwd_r_wps);
}

// tiles per dW item for a call with N nodes: the plan's value, lowered for small N when the dW_r kernel
// (one CTA per (item, 32-channel block), items processed serially) would otherwise be bound by its
// longest item: at most N / (64 x the CTA slots per channel block) nodes per item (148 SMs x 3 CTAs)
int tiles_per_item(const symcon_plan* p, int64_t N) {
  const int t = p->kc.dw_tiles_per_item;
  if (!p->kc.dw_r || p->t.simple || !p->kc.dw_items_adapt) return t;
  const int64_t slots = std::max<int64_t>(1, 148 * 3 / ((p->t.K + 31) / 32));
  const int64_t want = N / ((int64_t)p->kc.tile_nodes * slots);
  return (int)std::max<int64_t>(1, std::min<int64_t>(t, want));
}

WsLayout layout(const symcon_plan* p, int64_t N) {
  WsLayout w{};
  const size_t fs = esz(p);
  const int E = p->t.E, K = p->t.K;
  const size_t nch = bucket_chunks(N);
  w.max_tiles = N / p->kc.tile_nodes + E + 1;
  w.max_items = w.max_tiles / tiles_per_item(p, N) + E + 1;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  w.err = take(sizeof(unsigned long long));  // first: its offset must not depend on N
  w.hist = take(sizeof(int) * nch * (E + 1));
  w.chunk_bad = take(sizeof(int) * std::max<size_t>(nch, 1));
  w.off = take(sizeof(int) * nch * (E + 1));
  w.seg_off = take(sizeof(int) * (E + 2));
  w.perm = take(sizeof(int) * std::max<int64_t>(N, 1));
  w.tiles = take(sizeof(int4) * w.max_tiles);
  w.n_tiles = take(sizeof(int));
  w.items = take(sizeof(int4) * w.max_items);
  w.n_items = take(sizeof(int));
  w.item_off = take(sizeof(int) * (E + 2));
  w.tile_off = take(sizeof(int) * (E + 2));
  w.tile_perm = take(sizeof(int) * (size_t)w.max_tiles * p->kc.tile_nodes);
  w.coef = take(fs * (size_t)E * K * p->npad);
  w.spart = take(fs * (size_t)w.max_items * K * p->npad * (p->kc.dw_r ? p->kc.dw_r_wps : 1));   // dw_r_wps partials per item
  w.stot = take(fs * (size_t)E * K * p->npad);
  w.coef_r = take(sizeof(float) * (size_t)E * p->t.out_per_ch * p->kc.fwd_r_split * std::max(p->rnq, 1) * K * 4);
  w.dw_count = take(sizeof(int) * (size_t)E * ((K + 31) / 32));
  w.coef2 = take(sizeof(float) * (size_t)E * K * p->npad);   // the uW fold of the double backward
  w.coef_r2 = take(sizeof(float) * (size_t)E * p->t.out_per_ch * p->kc.fwd_r_split * std::max(p->rnq, 1) * K * 4);
  w.total = o;
  return w;
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
  return h;
}

std::string lib_dir() {
  Dl_info info;
  if (dladdr((void*)&symcon_status_string, &info) && info.dli_fname) {
    std::string f = info.dli_fname;
    auto pos = f.rfind('/');
    if (pos != std::string::npos) return f.substr(0, pos);
  }
  return ".";
}

std::string cache_dir() {
  const char* e = getenv("SYMCON_KCACHE");
  std::string d = e && *e ? e : lib_dir() + "/_kcache";
  mkdir(d.c_str(), 0775);
  return d;
}

const std::vector<std::string>& nvrtc_opts() {
  static std::vector<std::string> o = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17",
                                       "--ptxas-options=-v", "-DSYMCON_GENERATED=1"};
  return o;
}

std::mutex g_compile_mu;

// returns cubin bytes; compiles with NVRTC and caches on disk
bool get_cubin(const std::string& src, std::vector<char>& cubin, std::string* path_out) {
  std::string key = src;
  for (auto& s : nvrtc_opts()) key += "\n" + s;
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  key += "\nnvrtc" + std::to_string(maj) + "." + std::to_string(min);
  char name[64];
  snprintf(name, sizeof name, "symcon_%016llx", (unsigned long long)fnv1a(key));
  std::string dir = cache_dir();
  std::string path = dir + "/" + name + ".cubin";
  if (path_out) *path_out = path;
  std::lock_guard<std::mutex> g(g_compile_mu);
  {
    std::ifstream f(path, std::ios::binary);
    if (f) {
      cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
      if (!cubin.empty()) return true;
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "symcon_generated.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    set_error("nvrtcCreateProgram failed");
    return false;
  }
  std::vector<const char*> opts;
  for (auto& s : nvrtc_opts()) opts.push_back(s.c_str());
  nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  size_t logsz = 0;
  nvrtcGetProgramLogSize(prog, &logsz);
  std::string log(logsz, '\0');
  if (logsz) nvrtcGetProgramLog(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    set_error("NVRTC compile failed: " + log.substr(0, 4000));
    std::ofstream(dir + "/" + name + ".failed.cu") << src;
    nvrtcDestroyProgram(&prog);
    return false;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.resize(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  std::string tmp = path + ".tmp" + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    f.write(cubin.data(), (std::streamsize)cubin.size());
  }
  rename(tmp.c_str(), path.c_str());
  std::ofstream(dir + "/" + name + ".log") << log;
  std::ofstream(dir + "/" + name + ".cu") << src;
  return true;
}

symcon_status cuda_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SYMCON_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SYMCON_ECUDA;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

symcon_status validate_build(int lmax_in, int corr, const int* out_L, int n_out, int E, int K) {
  if (lmax_in < 0 || lmax_in > 3) { set_error("lmax_in must be in [0,3]"); return SYMCON_EINVAL; }
  if (corr < 1) { set_error("correlation must be >= 1"); return SYMCON_EINVAL; }
  if (corr > 4) { set_error("correlation must be <= 4"); return SYMCON_EUNSUPPORTED; }
  if (!out_L || n_out < 1 || n_out > 4) { set_error("n_out must be in [1,4]"); return SYMCON_EINVAL; }
  for (int i = 0; i < n_out; i++) {
    if (out_L[i] < 0 || out_L[i] > 3) { set_error("out_L values must be in [0,3]"); return SYMCON_EINVAL; }
    if (i && out_L[i] <= out_L[i - 1]) { set_error("out_L must be strictly increasing"); return SYMCON_EINVAL; }
  }
  if (E < 1 || E > 8192) { set_error("num_elements must be in [1, 8192]"); return SYMCON_EINVAL; }
  if (K < 1 || K > (1 << 20)) { set_error("channels must be >= 1"); return SYMCON_EINVAL; }
  return SYMCON_OK;
}

}  // namespace

namespace symcon {
bool compile_cubin(const std::string& src, std::vector<char>& cubin) { return get_cubin(src, cubin, nullptr); }
symcon_status cuda_status(cudaError_t e, const char* what) { return cuda_err(e, what); }
}  // namespace symcon

extern "C" {

const char* symcon_status_string(symcon_status s) {
  switch (s) {
    case SYMCON_OK: return "ok";
    case SYMCON_EINVAL: return "invalid argument";
    case SYMCON_EUNSUPPORTED: return "unsupported";
    case SYMCON_ECUDA: return "CUDA error";
    case SYMCON_ENOMEM: return "out of memory / workspace too small";
    case SYMCON_EELEMENT: return "node_elem out of range (species index without weights)";
    case SYMCON_ETIMEOUT: return "peer all-reduce barrier timed out";
  }
  return "unknown";
}

const char* symcon_last_error(void) { return g_last_error.c_str(); }

symcon_status symcon_real_cg(int l1, int l2, int L, double* out) {
  if (!out || l1 < 0 || l2 < 0 || L < 0 || l1 > 3 || l2 > 3 || L > 6) { set_error("bad l"); return SYMCON_EINVAL; }
  auto c = real_coupling(l1, l2, L);
  std::memcpy(out, c.data(), c.size() * sizeof(double));
  return SYMCON_OK;
}

static symcon_status build_common(int lmax_in, int corr, const int* out_L, int n_out, int E, int K, symcon_plan** out,
                                  int dtype = SYMCON_F32) {
  symcon_status s = validate_build(lmax_in, corr, out_L, n_out, E, K);
  if (s) return s;
  auto* p = new (std::nothrow) symcon_plan();
  if (!p) return SYMCON_ENOMEM;
  if (!parse_kernel_config(getenv("SYMCON_KCONFIG"), p->kc) || p->kc.node_pairs_per_lane < 1 ||
      p->kc.node_pairs_per_lane > 2) {
    set_error("bad SYMCON_KCONFIG");
    delete p;
    return SYMCON_EINVAL;
  }
  p->kc.tile_nodes = 64 * p->kc.node_pairs_per_lane;
  // dW items: ~256 nodes
  if (p->kc.node_pairs_per_lane == 2 && p->kc.dw_tiles_per_item == 4) p->kc.dw_tiles_per_item = 2;
  std::vector<int> ol(out_L, out_L + n_out);
  if (!build_tables(lmax_in, corr, ol, E, K, p->t)) { delete p; return SYMCON_EINVAL; }
  p->npad = (int)((p->t.rows.size() + 31) / 32 * 32);
  p->t.f64 = dtype == SYMCON_F64;
  p->t.simple = p->t.f64 || corr == 4;
  // measured defaults (profiles/r01): few large row groups when the dB row is short (MP-medium:
  // 52 rows x 8 warps, fewer smem reads per FMA), smaller groups for the 9-output large shape
  if (p->kc.dw_rows_per_group <= 0) p->kc.dw_rows_per_group = p->t.out_per_ch > 4 ? 56 : 52;
  if (p->kc.dw_groups_per_cta <= 0) p->kc.dw_groups_per_cta = 8;
  // q-form dW measured 6% faster at 9 outputs per channel (large), 1.5% slower at 4 (MP-medium)
  if (p->kc.dw_qform < 0) p->kc.dw_qform = p->t.out_per_ch > 4 ? 1 : 0;
  // gamma kernels (bit 1: forward, bit 2: dA): measured on the OFF-small shape, the gamma dA is
  // 16% faster than the persistent one and the gamma forward 27% slower -> auto = dA only
  if (p->kc.gamma < 0) p->kc.gamma = p->t.rows.size() <= 128 ? 2 : 0;
  // W_bar also holds the JVP direction rows in registers: at most 8 warps (255 registers each)
  // (and enough warps that the register staging of A, U and dB stays small)
  if (p->kc.dw2_rows_per_group <= 0) {
    const int nrows = (int)p->t.rows.size();
    p->kc.dw2_rows_per_group = p->t.out_per_ch > 4 ? 40 : std::min(52, std::max(16, (nrows + 7) / 8));
  }
  if (p->kc.dw2_groups_per_cta <= 0) p->kc.dw2_groups_per_cta = 8;
  // measured (profiles/r02): fwd_r beats symcon_fwd at 1 and 4 output slots (OFF-small, MP-medium) and
  // loses at 9 (large: 9 warps x 166 registers per CTA)
  if (p->kc.fwd_r < 0) p->kc.fwd_r = p->t.out_per_ch <= 4 ? 1 : 0;
  if (p->kc.fold_split < 1 || p->kc.fold_split > 16) { set_error("bad fold_split"); delete p; return SYMCON_EINVAL; }
  if (p->kc.fwd_r_nst < 2 || p->kc.fwd_r_nst > 8 || p->kc.dw_r_nst < 2 || p->kc.dw_r_nst > 8) { set_error("bad ring depth"); delete p; return SYMCON_EINVAL; }
  if (p->kc.fwd_r_tr) { set_error("fwd_r_tr is not available with the mbarrier ring"); delete p; return SYMCON_EINVAL; }
  if (p->kc.fwd_r_block < 2 || p->kc.fwd_r_block > 32 || (p->kc.fwd_r_block & 1) || 64 % p->kc.fwd_r_block) {
    set_error("bad fwd_r_block");
    delete p;
    return SYMCON_EINVAL;
  }
  if (p->kc.fwd_r && !p->t.simple) {
    if (p->kc.fwd_r_split != 1 && (p->kc.fwd_r_split != 2 || p->kc.fwd_r_npw != 1)) { set_error("fwd_r_split must be 1 or 2 (with fwd_r_npw 1)"); delete p; return SYMCON_EINVAL; }
    // measured (profiles/r02): with one output slot (OFF-small) a 1-warp CTA leaves 3 warps per SM;
    // 4 warps sharing each stage's node pairs cut the forward 0.051 -> 0.036 ms
    if (p->kc.fwd_r_wps <= 0) p->kc.fwd_r_wps = p->t.out_per_ch == 1 ? 4 : 1;
    if (p->kc.fwd_r_split > 1) p->kc.fwd_r_wps = 1;
    // slot groups (several CTAs per node block): auto 3 at 9 slots (large) -> 3 warps per CTA
    if (p->kc.fwd_r_groups <= 0) p->kc.fwd_r_groups = (p->t.out_per_ch > 4 && p->t.out_per_ch % 3 == 0) ? 3 : 1;
    if (p->kc.fwd_r_split > 1 || (p->t.out_per_ch * p->kc.fwd_r_split) % p->kc.fwd_r_groups) p->kc.fwd_r_groups = 1;
    if (p->kc.fwd_r_wps < 1 || p->kc.fwd_r_wps * p->kc.fwd_r_npw > p->kc.fwd_r_block / 2) { set_error("bad fwd_r_wps"); delete p; return SYMCON_EINVAL; }
    for (auto& h : horner_vslots(p->t, p->kc.fwd_r_split)) p->rnq = std::max(p->rnq, (int)((h.rows.size() + 3) / 4));
    if (p->t.n_lm != 16) p->kc.fwd_r = 0;   // the A staging is laid out for 16 floats per (node, channel) (lmax_in 3)
  }
  // measured (profiles/r02): dW_r -22% at MP-medium (4 slots), OFF-small (1 slot) step 0.154 vs 0.196 ms,
  // large (9 slots, as 3 row-group sets) dW 4.84 vs 5.97 ms (with dA after dW, dist.DataParallelContraction)
  if (p->kc.dw_r < 0) p->kc.dw_r = 1;
  // dw_r stages 16-byte chunks of A rows (16 floats at lmax_in 3) and of 32-channel dB slices
  // (K % 32 != 0 falls back to symcon_bwd_dW at load time; the source does not depend on K)
  if (p->t.n_lm != 16) p->kc.dw_r = 0;
  if (p->kc.da_s < 0) p->kc.da_s = 0;
  if (p->kc.dw_r_block < 2 || 64 % p->kc.dw_r_block) { set_error("bad dw_r_block"); delete p; return SYMCON_EINVAL; }
  // dW_r warps per slot: measured at OFF-small (1 slot) the dW kernel alone is faster with 2 (0.042 vs
  // 0.051 ms) but the step slower (0.186 vs 0.154 ms: less room for the concurrent dA) -> auto 1;
  // at most 16 warps per CTA
  if (p->kc.dw_r_wps <= 0) p->kc.dw_r_wps = 1;
  // dW_r row-group sets (grid.z): auto 3 at 9 slots (large), so a CTA holds 3 slot warps
  if (p->kc.dw_r_groups <= 0) p->kc.dw_r_groups = (p->t.out_per_ch > 4 && p->t.out_per_ch % 3 == 0) ? 3 : 1;
  if (p->kc.dw_r_fuse || (p->t.out_per_ch * std::max(1, p->kc.dw_r_split)) % p->kc.dw_r_groups) p->kc.dw_r_groups = 1;
  if (32 * p->t.out_per_ch * std::max(1, p->kc.dw_r_split) * p->kc.dw_r_wps > 512 * std::max(1, p->kc.dw_r_groups)) p->kc.dw_r_wps = 1;
  if (p->kc.dw_r_wps > p->kc.dw_r_block) { set_error("bad dw_r_wps"); delete p; return SYMCON_EINVAL; }
  if (p->kc.dw_r_wps > 1) { p->kc.unfold_reduce = 0; p->kc.dw_r_fuse = 0; }
  if (p->t.simple) {   // fp64 or correlation 4: the plain scalar kernels of codegen_simple.cpp
    p->kc.fwd_r = p->kc.dw_r = p->kc.da_s = 0;
    p->kc.gamma = 0;
    // table-driven fold / unfold: split rows / columns over grid.z (~256 per CTA)
    p->kc.fold_split = std::min(16, std::max(1, p->npad / 256));
    p->kc.simple_unfold_split = std::min(16, std::max(1, (int)p->t.paths.size() / 64));
    // dW rows per warp: fewer row groups = fewer re-reads of each node's A row; measured (profiles/r02):
    // fp64 MP-medium dW 1.63 ms at 96 vs 2.68 ms at 48 (128 spills); correlation 4 fp32 2.84 ms at 128
    // vs 5.97 ms at 48 (192: same as 128)
    if (p->kc.simple_rpg <= 0) p->kc.simple_rpg = p->t.f64 ? 96 : 128;
    // coefficient rows of the SWPC warps of a fwd / dA CTA in dynamic shared memory (<= 200 KB)
    const size_t row_bytes = esz(p) * (size_t)p->npad;
    p->kc.simple_warps = 4;
    while (p->kc.simple_warps > 1 && row_bytes * p->kc.simple_warps > 200 * 1024) p->kc.simple_warps--;
    if (row_bytes > 200 * 1024) { set_error("folded table too large for shared memory"); delete p; return SYMCON_EUNSUPPORTED; }
    p->simple_smem = row_bytes * p->kc.simple_warps;

    p->kc.unfold_reduce = 0;
    p->source = generate_source_simple(p->t, p->kc);
  } else {
    p->source = generate_source(p->t, p->kc);
  }
  *out = p;
  return SYMCON_OK;
}

symcon_status symcon_build_tables(int lmax_in, int correlation, const int* out_L, int n_out, int num_elements,
                                  int channels, int device, symcon_plan** plan) {
  return symcon_build_tables_ex(lmax_in, correlation, out_L, n_out, num_elements, channels, device, SYMCON_F32, plan);
}

symcon_status symcon_build_tables_ex(int lmax_in, int correlation, const int* out_L, int n_out, int num_elements,
                                     int channels, int device, int32_t dtype, symcon_plan** plan) {
  if (!plan) { set_error("plan is NULL"); return SYMCON_EINVAL; }
  *plan = nullptr;
  if (dtype != SYMCON_F32 && dtype != SYMCON_F64) { set_error("dtype must be SYMCON_F32 or SYMCON_F64"); return SYMCON_EINVAL; }
  symcon_plan* p = nullptr;
  symcon_status s = build_common(lmax_in, correlation, out_L, n_out, num_elements, channels, &p, dtype);
  if (s) return s;
  p->device = device;
  if (device >= 0) {
    int ndev = 0;
    if ((s = cuda_err(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount"))) { delete p; return s; }
    if (device >= ndev) { set_error("device out of range"); delete p; return SYMCON_EINVAL; }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    int maj = 0, mnr = 0;
    cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, device);
    if (maj != 10 || mnr != 0) {
      set_error("libsymcon kernels are built for sm_100a (B200); device is sm_" + std::to_string(maj) + std::to_string(mnr));
      cudaSetDevice(prev);
      delete p;
      return SYMCON_EUNSUPPORTED;
    }
    std::vector<char> cubin;
    if (!get_cubin(p->source, cubin, nullptr)) { cudaSetDevice(prev); delete p; return SYMCON_ECUDA; }
    s = cuda_err(cudaLibraryLoadData(&p->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0), "cudaLibraryLoadData");
    if (!s && p->kc.fold_fork) {
      s = cuda_err(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking), "aux stream");
      if (!s) s = cuda_err(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "fork event");
      if (!s) s = cuda_err(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming), "join event");
    }
    if (!s && p->t.simple) {   // simple plan: fold, fwd, dA, dW, reduce_simple, unfold (codegen_simple.cpp)
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_fold, p->lib, "symcon_fold"), "get symcon_fold");
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_fwd, p->lib, "symcon_fwd"), "get symcon_fwd");
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_dA, p->lib, "symcon_bwd_dA"), "get symcon_bwd_dA");
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_dW, p->lib, "symcon_bwd_dW"), "get symcon_bwd_dW");
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_unfold, p->lib, "symcon_unfold"), "get symcon_unfold");
      if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_reduce_s, p->lib, "symcon_reduce_simple"), "get symcon_reduce_simple");
      int sms = 0, occ_f = 0, occ_a = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      const int nthr = 32 * p->kc.simple_warps;
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->simple_smem, device),
                           "smem fwd");
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_dA, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->simple_smem, device),
                           "smem dA");
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, (const void*)p->k_fwd, nthr, p->simple_smem), "occupancy fwd");
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, (const void*)p->k_dA, nthr, p->simple_smem), "occupancy dA");
      p->grid_fwd = sms * std::max(occ_f, 1);
      p->grid_dA = sms * std::max(occ_a, 1);
      cudaSetDevice(prev);
      if (s) { if (p->lib) cudaLibraryUnload(p->lib); delete p; return s; }
      *plan = p;
      return SYMCON_OK;
    }
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_fold, p->lib, "symcon_fold"), "get symcon_fold");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_fwd, p->lib, "symcon_fwd"), "get symcon_fwd");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_dA, p->lib, "symcon_bwd_dA"), "get symcon_bwd_dA");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_dW, p->lib, "symcon_bwd_dW"), "get symcon_bwd_dW");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_unfold, p->lib, "symcon_unfold"), "get symcon_unfold");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_bwd2, p->lib, "symcon_bwd2"), "get symcon_bwd2");
    if (!s) s = cuda_err(cudaLibraryGetKernel(&p->k_bwd2_dW, p->lib, "symcon_bwd2_dW"), "get symcon_bwd2_dW");
    if (!s && (p->kc.gamma & 1)) s = cuda_err(cudaLibraryGetKernel(&p->k_fwd_g, p->lib, "symcon_fwd_g"), "get symcon_fwd_g");
    if (!s && (p->kc.gamma & 2)) s = cuda_err(cudaLibraryGetKernel(&p->k_dA_g, p->lib, "symcon_bwd_dA_g"), "get symcon_bwd_dA_g");
    if (!s && p->k_dA_g) {
      int occ = 0, sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->k_dA_g, 128, 0), "occupancy dA_g");
      p->warp_slots_dA_g = sms * std::max(occ, 1) * 4;
    }
    if (!s && p->kc.fwd_r) {
      s = cuda_err(cudaLibraryGetKernel(&p->k_fwd_r, p->lib, "symcon_fwd_r"), "get symcon_fwd_r");
      p->fwd_r_smem = sizeof(float) * p->kc.fwd_r_nst * (size_t)p->kc.fwd_r_block * 512 + 16 * p->kc.fwd_r_nst +
                      sizeof(int) * p->kc.fwd_r_nst * (size_t)p->kc.fwd_r_block;
      if (p->kc.fwd_r_tr) p->fwd_r_smem += sizeof(float) * (size_t)p->kc.fwd_r_block * 512 + 64;   // the interleaved copy
      if (p->kc.fwd_r_split > 1) p->fwd_r_smem += 8 + sizeof(unsigned long long) * 2 * p->t.out_per_ch * 32;   // half-slot partials
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_fwd_r, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)p->fwd_r_smem, device), "fwd_r smem attribute");
      int sms = 0, occ = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->k_fwd_r, fwd_r_threads(p),
                                                                         p->fwd_r_smem), "occupancy fwd_r");
      if (p->kc.fwd_r_ctas_per_sm > 0) occ = std::min(occ, p->kc.fwd_r_ctas_per_sm);
      p->grid_fwd_r = sms * std::max(occ, 1);
      p->grid_fwd_r -= p->grid_fwd_r % std::max(1, p->kc.fwd_r_groups);   // whole slot groups
    }
    if (!s && p->kc.da_s) {
      s = cuda_err(cudaLibraryGetKernel(&p->k_dA_s, p->lib, "symcon_bwd_dA_s"), "get symcon_bwd_dA_s");
      p->da_s_smem = sizeof(float) * (size_t)p->kc.da_s_warps * 2 * p->npad;
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_dA_s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)p->da_s_smem, device), "dA_s smem attribute");
      int sms = 0, occ = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->k_dA_s, 32 * p->kc.da_s_warps,
                                                                         p->da_s_smem), "occupancy dA_s");
      p->grid_dA_s = sms * std::max(occ, 1);
    }
    if (!s && p->kc.dw_r && p->t.K % 32 == 0) {
      s = cuda_err(cudaLibraryGetKernel(&p->k_dW_r, p->lib, "symcon_bwd_dW_r"), "get symcon_bwd_dW_r");
      size_t dbw = 0;
      for (int L : p->t.out_L) dbw += 32 * (2 * L + 1);
      p->dw_r_smem = sizeof(float) * p->kc.dw_r_nst * (size_t)p->kc.dw_r_block * (512 + dbw) + 16 * p->kc.dw_r_nst +
                     sizeof(int) * (p->kc.dw_r_nst * (size_t)p->kc.dw_r_block + 1);
      // the S table of the fused reduction / the single-item unfold aliases the ring (same condition as the
      // codegen's: with row-group sets a CTA never unfolds, and must not pay the larger smem)
      const bool unf1 = p->kc.dw_r_unfold_single && p->kc.dw_r_wps == 1 && p->kc.dw_r_groups == 1 && !p->kc.dw_r_fuse &&
                        !p->kc.unfold_reduce;
      if (p->kc.dw_r_fuse || unf1)
        p->dw_r_smem = std::max(p->dw_r_smem, sizeof(float) * (size_t)p->npad * 33);
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_dW_r, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)p->dw_r_smem, device), "dW_r smem attribute");
    }
    p->tile_smem = sizeof(float) * (size_t)p->kc.tile_warps * (2 * (size_t)p->npad) + 16 * (size_t)p->kc.tile_warps;
    if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)p->tile_smem, device), "fwd smem attribute");
    if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_dA, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)p->tile_smem, device), "dA smem attribute");
    if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_bwd2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)p->tile_smem, device), "bwd2 smem attribute");
    if (!s) {
      int sms = 0, occ_f = 0, occ_a = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, (const void*)p->k_fwd, 32 * p->kc.tile_warps,
                                                                 p->tile_smem), "occupancy fwd");
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, (const void*)p->k_dA, 32 * p->kc.tile_warps,
                                                                         p->tile_smem), "occupancy dA");
      int occ_2 = 0;
      if (!s) s = cuda_err(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_2, (const void*)p->k_bwd2, 32 * p->kc.tile_warps,
                                                                         p->tile_smem), "occupancy bwd2");
      p->grid_bwd2 = sms * std::max(occ_2, 1);
      p->grid_fwd = sms * std::max(occ_f, 1);
      p->grid_dA = std::max(1, sms - std::max(0, p->kc.da_reserve_sms)) *
                   std::max(p->kc.da_ctas_per_sm > 0 ? std::min(occ_a, p->kc.da_ctas_per_sm) : occ_a, 1);
    }
    {
      const int nout = p->t.out_per_ch, nrows = (int)p->t.rows.size();
      const int ng = (nrows + p->kc.dw_rows_per_group - 1) / p->kc.dw_rows_per_group;  // must match codegen
      p->dw_nz = (ng + p->kc.dw_groups_per_cta - 1) / p->kc.dw_groups_per_cta;
      p->dw_gpc = (ng + p->dw_nz - 1) / p->dw_nz;
      const int ng2 = (nrows + p->kc.dw2_rows_per_group - 1) / p->kc.dw2_rows_per_group;
      p->dw2_nz = (ng2 + p->kc.dw2_groups_per_cta - 1) / p->kc.dw2_groups_per_cta;
      p->dw2_gpc = (ng2 + p->dw2_nz - 1) / p->dw2_nz;
      p->dw_smem = sizeof(float) * (size_t)p->kc.dw_block_nodes * (p->t.n_lm + nout) * 34;
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_dW, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)p->dw_smem, device), "dW smem attribute");
      p->dw2_smem = sizeof(float) * (size_t)p->kc.dw_block_nodes * (2 * p->t.n_lm + nout) * 34;
      if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_bwd2_dW, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)p->dw2_smem, device), "bwd2_dW smem attribute");
    }
    p->unfold_smem = sizeof(float) * 32 * (size_t)(p->npad + 1);
    if (!s) s = cuda_err(cudaKernelSetAttributeForDevice(p->k_unfold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)p->unfold_smem, device), "unfold smem attribute");
    cudaSetDevice(prev);
    if (s) { if (p->lib) cudaLibraryUnload(p->lib); delete p; return s; }
  }
  *plan = p;
  return SYMCON_OK;
}

/* Compile (NVRTC, sm_100a) the kernels for a configuration into the cubin cache without a
 * device (used by the build step on CPU-only hosts). Writes the cubin path if path != NULL. */
symcon_status symcon_precompile(int lmax_in, int correlation, const int* out_L, int n_out, char* path, size_t path_len) {
  return symcon_precompile_ex(lmax_in, correlation, out_L, n_out, SYMCON_F32, path, path_len);
}

symcon_status symcon_precompile_ex(int lmax_in, int correlation, const int* out_L, int n_out, int32_t dtype, char* path,
                                   size_t path_len) {
  symcon_plan* p = nullptr;
  symcon_status s = build_common(lmax_in, correlation, out_L, n_out, 1, 1, &p, dtype);
  if (s) return s;
  std::vector<char> cubin;
  std::string cp;
  bool ok = get_cubin(p->source, cubin, &cp);
  delete p;
  if (!ok) return SYMCON_ECUDA;
  if (path && path_len) { strncpy(path, cp.c_str(), path_len - 1); path[path_len - 1] = 0; }
  return SYMCON_OK;
}

/* Copy the generated CUDA source of a plan (NULL buf: returns the needed size incl. NUL). */
size_t symcon_plan_source(const symcon_plan* p, char* buf, size_t len) {
  if (!p) return 0;
  if (!buf) return p->source.size() + 1;
  size_t n = std::min(len - 1, p->source.size());
  memcpy(buf, p->source.data(), n);
  buf[n] = 0;
  return n + 1;
}

symcon_status symcon_plan_info(const symcon_plan* p, symcon_info* info) {
  if (!p || !info) { set_error("NULL argument"); return SYMCON_EINVAL; }
  memset(info, 0, sizeof *info);
  const Tables& t = p->t;
  info->lmax_in = t.lmax_in;
  info->correlation = t.corr;
  info->n_out = (int)t.out_L.size();
  info->num_elements = t.E;
  info->channels = t.K;
  for (size_t i = 0; i < t.out_L.size(); i++) info->out_L[i] = t.out_L[i];
  for (auto& pd : t.paths) {
    int oi = (int)(std::find(t.out_L.begin(), t.out_L.end(), pd.L) - t.out_L.begin());
    info->eta[oi][pd.nu - 1]++;
  }
  info->n_paths = (int64_t)t.paths.size();
  info->weight_numel = (int64_t)t.E * info->n_paths * t.K;
  info->in_dim = (int64_t)t.K * t.n_lm;
  info->out_dim = (int64_t)t.K * t.out_per_ch;
  info->n_raw_terms = t.n_raw_terms;
  info->n_sym_terms = t.n_sym_terms;
  info->n_fold = (int64_t)t.rows.size();
  info->n_monomials = t.n_monomials;
  info->device = p->device;
  info->reserved = p->t.f64 ? SYMCON_F64 : SYMCON_F32;   // dtype
  return SYMCON_OK;
}

symcon_status symcon_plan_path(const symcon_plan* p, int64_t col, int32_t* L, int32_t* nu, int32_t* eta,
                               int32_t* ls, int32_t* mids) {
  if (!p || col < 0 || col >= (int64_t)p->t.paths.size()) { set_error("bad column"); return SYMCON_EINVAL; }
  const PathDesc& d = p->t.paths[col];
  if (L) *L = d.L;
  if (nu) *nu = d.nu;
  if (eta) *eta = d.eta;
  if (ls) for (int j = 0; j < d.nu; j++) ls[j] = d.ls[j];
  if (mids) for (int j = 0; j + 1 < d.nu; j++) mids[j] = d.mids[j];
  return SYMCON_OK;
}

static symcon_status sym_table(const symcon_plan* p, int64_t* n, int32_t* L, int32_t* M, int32_t* mono, int nm, int32_t* col,
                               double* value) {
  if (!p || !n) { set_error("NULL argument"); return SYMCON_EINVAL; }
  if (!L && !M && !mono && !col && !value) { *n = p->t.n_sym_terms; return SYMCON_OK; }
  if (mono && nm < p->t.corr) { set_error("correlation-4 plan: use symcon_plan_sym_table4"); return SYMCON_EUNSUPPORTED; }
  if (*n < p->t.n_sym_terms) { *n = p->t.n_sym_terms; set_error("arrays too small"); return SYMCON_ENOMEM; }
  int64_t q = 0;
  for (auto& r : p->t.rows)
    for (auto& cv : r.cols) {
      if (L) L[q] = r.L;
      if (M) M[q] = r.M;
      if (mono) for (int j = 0; j < nm; j++) mono[nm * q + j] = r.mono[j];
      if (col) col[q] = cv.first;
      if (value) value[q] = cv.second;
      q++;
    }
  *n = q;
  return SYMCON_OK;
}

symcon_status symcon_plan_sym_table(const symcon_plan* p, int64_t* n, int32_t* L, int32_t* M, int32_t* mono3,
                                    int32_t* col, double* value) {
  return sym_table(p, n, L, M, mono3, 3, col, value);
}

symcon_status symcon_plan_sym_table4(const symcon_plan* p, int64_t* n, int32_t* L, int32_t* M, int32_t* mono4,
                                     int32_t* col, double* value) {
  return sym_table(p, n, L, M, mono4, 4, col, value);
}

size_t symcon_workspace_bytes(const symcon_plan* p, int64_t N) {
  if (!p || N < 0) return 0;
  return layout(p, N).total;
}

int32_t symcon_last_launch_count(const symcon_plan* p) { return p ? p->last_launches.load() : 0; }

static symcon_status check_common(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                  void* ws, size_t ws_bytes) {
  if (!p) { set_error("plan is NULL"); return SYMCON_EINVAL; }
  if (p->device < 0 || !p->lib) { set_error("host-only plan: no kernels loaded"); return SYMCON_EINVAL; }
  if (N < 0 || N > (int64_t)0x7fffffff) { set_error("num_nodes out of range"); return SYMCON_EINVAL; }
  if (N == 0) return SYMCON_OK;
  if (!A || !W || !ne || !ws) { set_error("NULL device pointer"); return SYMCON_EINVAL; }
  if (!aligned16(A) || !aligned16(ws)) { set_error("A and workspace must be 16-byte aligned"); return SYMCON_EINVAL; }
  if (ws_bytes < layout(p, N).total) { set_error("workspace too small"); return SYMCON_ENOMEM; }
  return SYMCON_OK;
}

static void fill_params(const symcon_plan* p, const WsLayout& w, char* ws, int64_t N, Params& q) {
  memset(&q, 0, sizeof q);
  q.perm = (const int*)(ws + w.perm);
  q.tiles = (const int4*)(ws + w.tiles);
  q.n_tiles = (const int*)(ws + w.n_tiles);
  q.items = (const int4*)(ws + w.items);
  q.n_items = (const int*)(ws + w.n_items);
  q.item_off = (const int*)(ws + w.item_off);
  q.seg_off = (const int*)(ws + w.seg_off);
  q.coef = (float*)(ws + w.coef);
  q.spart = (float*)(ws + w.spart);
  q.tile_perm = (const int*)(ws + w.tile_perm);
  q.stot = (float*)(ws + w.stot);
  q.coef_r = (float*)(ws + w.coef_r);
  q.dw_count = (int*)(ws + w.dw_count);
  q.accum = 0;
  q.N = (int)N;
  q.K = p->t.K;
  q.E = p->t.E;
  q.zero = -0.0f;
}

static int launch_prep(const symcon_plan* p, const WsLayout& w, char* ws, int64_t N, const int32_t* ne, const float* W,
                       Params& q, cudaStream_t st, bool fold, symcon_status* s, uint32_t flags = 0) {
  int n = 0;
  bool skip_bucket = false, skip_fold = false;
  {
    std::lock_guard<std::mutex> g(p->ws_mu);
    auto& rec = p->ws_state[ws];
    skip_bucket = (flags & SYMCON_REUSE_BUCKETS) && rec.N == N && rec.ne == ne;
    skip_fold = (flags & SYMCON_REUSE_FOLD) && skip_bucket && rec.W == W;
    rec.N = N;
    rec.ne = ne;
    if (fold) rec.W = W;
  }
  if (skip_fold) fold = false;
  // the fold (W only) and the bucketing (node_elem only) are independent: fold on the plan's aux stream
  std::unique_lock<std::mutex> fork_lock(p->fork_mu, std::defer_lock);
  const bool fork = fold && !skip_bucket && p->aux;
  auto launch_fold = [&](cudaStream_t fs) {
    Timed tm(p, K_FOLD, fs);
    q.W = W;
    void* args[] = {&q};
    dim3 grid(p->t.E, (p->t.K + 31) / 32, p->kc.fold_split);
    *s = cuda_err(cudaLaunchKernel((const void*)p->k_fold, grid, dim3(128), args, 0, fs), "launch symcon_fold");
    n++;
  };
  if (fork) {
    fork_lock.lock();
    cudaEventRecord(p->ev_fork, st);
    cudaStreamWaitEvent(p->aux, p->ev_fork, 0);
    launch_fold(p->aux);
    cudaEventRecord(p->ev_join, p->aux);
    fold = false;
  }
  if (!skip_bucket) {
    BucketArgs b;
    b.node_elem = ne;
    b.N = (int)N;
    b.E = p->t.E;
    b.tile_nodes = p->kc.tile_nodes;
    b.tiles_per_item = tiles_per_item(p, N);
    b.hist = (int*)(ws + w.hist);
    b.off = (int*)(ws + w.off);
    b.seg_off = (int*)(ws + w.seg_off);
    b.perm = (int*)(ws + w.perm);
    b.tiles = (int4*)(ws + w.tiles);
    b.n_tiles = (int*)(ws + w.n_tiles);
    b.items = (int4*)(ws + w.items);
    b.n_items = (int*)(ws + w.n_items);
    b.item_off = (int*)(ws + w.item_off);
    b.err = (unsigned long long*)(ws + w.err);
    b.tile_off = (int*)(ws + w.tile_off);
    b.tile_perm = (int*)(ws + w.tile_perm);
    b.max_tiles = w.max_tiles;
    b.chunk_bad = (int*)(ws + w.chunk_bad);
    b.zero_buf = (int*)(ws + w.dw_count);
    b.zero_n = p->t.E * ((p->t.K + 31) / 32);
    b.fused = p->kc.bucket_fused;
    Timed tm(p, K_BUCKET, st);
    n += bucket_launch(b, st);
  }
  if (fork) {
    cudaStreamWaitEvent(st, p->ev_join, 0);
    fork_lock.unlock();
  }
  if (fold) launch_fold(st);
  return n;
}

// the forward kernel of the plan (fwd_r / gamma / persistent) with the coefficients q.coef(_r) already folded
static symcon_status launch_fwd_kernel(const symcon_plan* p, const WsLayout& w, Params& q, int64_t N, cudaStream_t st) {
  symcon_status s = SYMCON_OK;
  if (p->t.simple) {
    void* args[] = {&q};
    Timed tm(p, K_FWD, st);
    return cuda_err(cudaLaunchKernel((const void*)p->k_fwd, dim3(p->grid_fwd), dim3(32 * p->kc.simple_warps), args, p->simple_smem, st),
                    "launch symcon_fwd (simple)");
  }
  if (p->k_fwd_r && (s = encode_a_map(q.tmA, q.A, N, p->t.K, p->t.n_lm))) return s;
  void* args[] = {&q};
  Timed tm(p, K_FWD, st);
  if (p->k_fwd_r)
    return cuda_err(cudaLaunchKernel((const void*)p->k_fwd_r, dim3(p->grid_fwd_r), dim3(fwd_r_threads(p)), args, p->fwd_r_smem, st),
                    "launch symcon_fwd_r");
  if (p->k_fwd_g)
    return cuda_err(cudaLaunchKernel((const void*)p->k_fwd_g, dim3((unsigned)((w.max_tiles + 3) / 4), (p->t.K + 31) / 32), dim3(128),
                                     args, 0, st), "launch symcon_fwd_g");
  return cuda_err(cudaLaunchKernel((const void*)p->k_fwd, dim3(p->grid_fwd), dim3(32 * p->kc.tile_warps), args, p->tile_smem, st),
                  "launch symcon_fwd");
}

// the dA kernel of the plan (scalar / gamma / persistent)
static symcon_status launch_dA_kernel(const symcon_plan* p, const WsLayout& w, Params& q, cudaStream_t st) {
  void* args[] = {&q};
  Timed tm(p, K_DA, st);
  if (p->t.simple)
    return cuda_err(cudaLaunchKernel((const void*)p->k_dA, dim3(p->grid_dA), dim3(32 * p->kc.simple_warps), args, p->simple_smem, st),
                    "launch symcon_bwd_dA (simple)");
  if (p->k_dA_s)
    return cuda_err(cudaLaunchKernel((const void*)p->k_dA_s, dim3(p->grid_dA_s), dim3(32 * p->kc.da_s_warps), args, p->da_s_smem, st),
                    "launch symcon_bwd_dA_s");
  if (p->k_dA_g) {
    // warps split each tile's nodes (grid.z) when the tiles alone leave most warp slots empty
    const long long warps = (long long)w.max_tiles * ((p->t.K + 31) / 32);
    int split = p->kc.gamma_split;
    // measured at OFF-small: the step does not change with the split (dA runs concurrently with dW_r) -> auto 1
    if (split <= 0) split = 1;
    (void)warps;
    return cuda_err(cudaLaunchKernel((const void*)p->k_dA_g, dim3((unsigned)((w.max_tiles + 3) / 4), (p->t.K + 31) / 32, split), dim3(128),
                                     args, 0, st), "launch symcon_bwd_dA_g");
  }
  return cuda_err(cudaLaunchKernel((const void*)p->k_dA, dim3(p->grid_dA), dim3(32 * p->kc.tile_warps), args, p->tile_smem, st),
                  "launch symcon_bwd_dA");
}

static symcon_status forward_impl(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                  float* B, void* ws, size_t ws_bytes, void* stream);

symcon_status symcon_forward(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                             float* B, void* ws, size_t ws_bytes, void* stream) {
  if (p && p->t.f64) { set_error("fp64 plan: use symcon_forward_f64"); return SYMCON_EINVAL; }
  return forward_impl(p, N, A, W, ne, B, ws, ws_bytes, stream);
}

symcon_status symcon_forward_f64(const symcon_plan* p, int64_t N, const double* A, const double* W, const int32_t* ne,
                                 double* B, void* ws, size_t ws_bytes, void* stream) {
  if (p && !p->t.f64) { set_error("fp32 plan: use symcon_forward"); return SYMCON_EINVAL; }
  return forward_impl(p, N, (const float*)A, (const float*)W, ne, (float*)B, ws, ws_bytes, stream);
}

static symcon_status forward_impl(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                  float* B, void* ws, size_t ws_bytes, void* stream) {
  symcon_status s = check_common(p, N, A, W, ne, ws, ws_bytes);
  if (s) return s;
  p->last_launches = 0;
  if (N == 0) return SYMCON_OK;
  if (!B || !aligned16(B)) { set_error("B must be non-NULL and 16-byte aligned"); return SYMCON_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  WsLayout w = layout(p, N);
  Params q;
  fill_params(p, w, (char*)ws, N, q);
  q.A = A;
  q.W = W;
  q.node_elem = ne;
  q.B = B;
  int n = launch_prep(p, w, (char*)ws, N, ne, W, q, st, true, &s);
  if (s) return s;
  s = launch_fwd_kernel(p, w, q, N, st);
  n++;
  if (s) return s;
  p->last_launches = n;
  return cuda_err(cudaGetLastError(), "forward launch");
}

static symcon_status backward_impl(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                   const float* dB, float* dA, float* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                   void* stream);

symcon_status symcon_backward(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                              const float* dB, float* dA, float* dW, void* ws, size_t ws_bytes, void* stream) {
  return symcon_backward_ex(p, N, A, W, ne, dB, dA, dW, ws, ws_bytes, 0u, stream);
}

symcon_status symcon_backward_f64(const symcon_plan* p, int64_t N, const double* A, const double* W, const int32_t* ne,
                                  const double* dB, double* dA, double* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                  void* stream) {
  if (p && !p->t.f64) { set_error("fp32 plan: use symcon_backward_ex"); return SYMCON_EINVAL; }
  return backward_impl(p, N, (const float*)A, (const float*)W, ne, (const float*)dB, (float*)dA, (float*)dW, ws, ws_bytes,
                       flags, stream);
}

symcon_status symcon_backward_ex(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                 const float* dB, float* dA, float* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                 void* stream) {
  if (p && p->t.f64) { set_error("fp64 plan: use symcon_backward_f64"); return SYMCON_EINVAL; }
  return backward_impl(p, N, A, W, ne, dB, dA, dW, ws, ws_bytes, flags, stream);
}

static symcon_status backward_impl(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                   const float* dB, float* dA, float* dW, void* ws, size_t ws_bytes, uint32_t flags,
                                   void* stream) {
  if (!p) { set_error("plan is NULL"); return SYMCON_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  p->last_launches = 0;
  if (N == 0) {
    // no nodes: dW must still be overwritten with zeros (reading s12)
    if (dW) return cuda_err(cudaMemsetAsync(dW, 0, esz(p) * (size_t)p->t.E * p->t.paths.size() * p->t.K, st), "memset dW");
    return SYMCON_OK;
  }
  symcon_status s = check_common(p, N, A, W, ne, ws, ws_bytes);
  if (s) return s;
  if (!dB || !aligned16(dB)) { set_error("dB must be non-NULL and 16-byte aligned"); return SYMCON_EINVAL; }
  if (dA && !aligned16(dA)) { set_error("dA must be 16-byte aligned"); return SYMCON_EINVAL; }
  if (!dA && !dW) return SYMCON_OK;
  WsLayout w = layout(p, N);
  Params q;
  fill_params(p, w, (char*)ws, N, q);
  q.A = A;
  q.W = W;
  q.node_elem = ne;
  q.dB = dB;
  q.dA = dA;
  q.dW = dW;
  int n = launch_prep(p, w, (char*)ws, N, ne, W, q, st, dA != nullptr, &s, flags);
  if (s) return s;
  if (dW && p->k_dW_r && (s = encode_a_map(q.tmA, A, N, p->t.K, p->t.n_lm))) return s;
  // single-item elements finished (unfolded) by their dW_r CTA: the unfold kernel skips them
  q.pad = (dW && p->k_dW_r && p->kc.dw_r_unfold_single && p->kc.dw_r_wps == 1 && p->kc.dw_r_groups == 1 && !p->kc.dw_r_fuse &&
           !p->kc.unfold_reduce) ? 1 : 0;
  void* args[] = {&q};
  const unsigned ky = (p->t.K + p->kc.warps_per_cta - 1) / p->kc.warps_per_cta;
  if (dW && p->t.simple) {   // simple plans: S partials (item, row group, channel block), item reduction, unfold
    {
      Timed tm(p, K_DW, st);
      const int rpg = std::max(8, p->kc.simple_rpg), ng = ((int)p->t.rows.size() + rpg - 1) / rpg;   // = codegen_simple RPG
      s = cuda_err(cudaLaunchKernel((const void*)p->k_dW, dim3((unsigned)w.max_items, ng, (p->t.K + 31) / 32), dim3(32), args, 0, st),
                   "launch symcon_bwd_dW (simple)");
    }
    if (s) return s;
    Timed tm(p, K_UNFOLD, st);
    const long long per = (long long)p->npad * p->t.K;
    s = cuda_err(cudaLaunchKernel((const void*)p->k_reduce_s, dim3((unsigned)((per + 255) / 256), p->t.E), dim3(256), args, 0, st),
                 "launch symcon_reduce_simple");
    if (s) return s;
    s = cuda_err(cudaLaunchKernel((const void*)p->k_unfold, dim3(p->t.E, (p->t.K + 31) / 32, p->kc.simple_unfold_split), dim3(128),
                                  args, 0, st), "launch symcon_unfold (simple)");
    if (s) return s;
    n += 3;
  } else if (dW) {
    {
    Timed tm(p, K_DW, st);
    if (p->k_dW_r)   // S partials (+ with dw_r_fuse the element's item reduction and the unfold)
      s = cuda_err(cudaLaunchKernel((const void*)p->k_dW_r,
                                    dim3((unsigned)(w.max_items + (p->kc.dw_r_fuse ? p->t.E : 0)), p->t.K / 32, p->kc.dw_r_groups),
                                    dim3(32 * p->t.out_per_ch * std::max(1, p->kc.dw_r_split) / p->kc.dw_r_groups * p->kc.dw_r_wps), args,
                                    p->dw_r_smem, st),
                   "launch symcon_bwd_dW_r");
    else
      s = cuda_err(cudaLaunchKernel((const void*)p->k_dW, dim3((unsigned)(w.max_items * p->dw_nz), (p->t.K + 31) / 32, 1),
                                    dim3(32 * p->dw_gpc), args, p->dw_smem, st), "launch symcon_bwd_dW");
    }
    if (s) return s;
    if (!p->k_dW_r || !p->kc.dw_r_fuse) {
      Timed tm(p, K_UNFOLD, st);
      if (!p->kc.unfold_reduce)
        n += reduce_items_launch(q.spart, q.item_off, p->t.E, p->npad, p->t.K, q.stot, st,
                                 !p->k_dW_r ? 1 : (p->kc.dw_r_wps == 1 && !p->kc.dw_r_fuse) ? -1 : p->kc.dw_r_wps);
      s = cuda_err(cudaLaunchKernel((const void*)p->k_unfold, dim3(p->t.E, (p->t.K + 31) / 32), dim3(512), args,
                                    p->unfold_smem, st), "launch symcon_unfold");
      if (s) return s;
      n += 2;
    } else {
      n += 1;
    }
  }
  if (dA) {
    s = launch_dA_kernel(p, w, q, st);
    if (s) return s;
    n++;
  }
  p->last_launches = n;
  return cuda_err(cudaGetLastError(), "backward launch");
}

symcon_status symcon_backward2(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                               const float* dB, const float* uA, float* dB_bar, float* A_bar, float* W_bar, void* ws,
                               size_t ws_bytes, uint32_t flags, void* stream) {
  return symcon_backward2_ex(p, N, A, W, ne, dB, uA, nullptr, dB_bar, A_bar, W_bar, ws, ws_bytes, flags, stream);
}

symcon_status symcon_backward2_ex(const symcon_plan* p, int64_t N, const float* A, const float* W, const int32_t* ne,
                                  const float* dB, const float* uA, const float* uW, float* dB_bar, float* A_bar, float* W_bar,
                                  void* ws, size_t ws_bytes, uint32_t flags, void* stream) {
  if (!p) { set_error("plan is NULL"); return SYMCON_EINVAL; }
  if (p->t.simple) { set_error("the double backward is fp32 with correlation <= 3 only"); return SYMCON_EUNSUPPORTED; }
  cudaStream_t st = (cudaStream_t)stream;
  p->last_launches = 0;
  if (N == 0) {
    if (W_bar) return cuda_err(cudaMemsetAsync(W_bar, 0, sizeof(float) * (size_t)p->t.E * p->t.paths.size() * p->t.K, st), "memset W_bar");
    return SYMCON_OK;
  }
  symcon_status s = check_common(p, N, A, W, ne, ws, ws_bytes);
  if (s) return s;
  if (!dB || !aligned16(dB)) { set_error("dB must be non-NULL and 16-byte aligned"); return SYMCON_EINVAL; }
  if (!uA && !uW) { set_error("uA and uW are both NULL"); return SYMCON_EINVAL; }
  if (uA && !aligned16(uA)) { set_error("uA must be 16-byte aligned"); return SYMCON_EINVAL; }
  if ((dB_bar && !aligned16(dB_bar)) || (A_bar && !aligned16(A_bar))) {
    set_error("dB_bar and A_bar must be 16-byte aligned");
    return SYMCON_EINVAL;
  }
  if (!dB_bar && !A_bar && !W_bar) return SYMCON_OK;
  WsLayout w = layout(p, N);
  Params q;
  fill_params(p, w, (char*)ws, N, q);
  q.A = A;
  q.W = W;
  q.node_elem = ne;
  q.dB = dB;
  q.U = uA;
  q.B = dB_bar;
  q.dA = A_bar;
  q.dW = W_bar;
  const bool tile = dB_bar || A_bar;
  int n = launch_prep(p, w, (char*)ws, N, ne, W, q, st, tile, &s, flags);
  if (s) return s;
  void* args[] = {&q};
  if (!uA) {   // only the uW terms: start from zero
    if (W_bar && (s = cuda_err(cudaMemsetAsync(W_bar, 0, sizeof(float) * (size_t)p->t.E * p->t.paths.size() * p->t.K, st), "memset W_bar")))
      return s;
    if (dB_bar && (s = cuda_err(cudaMemsetAsync(dB_bar, 0, sizeof(float) * (size_t)N * p->t.K * p->t.out_per_ch, st), "memset dB_bar")))
      return s;
    if (A_bar && (s = cuda_err(cudaMemsetAsync(A_bar, 0, sizeof(float) * (size_t)N * p->t.K * p->t.n_lm, st), "memset A_bar")))
      return s;
  }
  if (W_bar && uA) {
    {
      Timed tm(p, K_BWD2_DW, st);
      s = cuda_err(cudaLaunchKernel((const void*)p->k_bwd2_dW, dim3((unsigned)(w.max_items * p->dw2_nz), (p->t.K + 31) / 32, 1),
                                    dim3(32 * p->dw2_gpc), args, p->dw2_smem, st), "launch symcon_bwd2_dW");
    }
    if (s) return s;
    Timed tm(p, K_UNFOLD, st);
    if (!p->kc.unfold_reduce) n += reduce_items_launch(q.spart, q.item_off, p->t.E, p->npad, p->t.K, q.stot, st);
    s = cuda_err(cudaLaunchKernel((const void*)p->k_unfold, dim3(p->t.E, (p->t.K + 31) / 32), dim3(512), args,
                                  p->unfold_smem, st), "launch symcon_unfold");
    if (s) return s;
    n += 2;
  }
  if (tile && uA) {
    {
      Timed tm(p, K_BWD2, st);
      s = cuda_err(cudaLaunchKernel((const void*)p->k_bwd2, dim3(p->grid_bwd2), dim3(32 * p->kc.tile_warps), args, p->tile_smem, st),
                   "launch symcon_bwd2");
    }
    if (s) return s;
    n++;
  }
  if (tile && uW) {
    // the cotangent uW of dW: dB_bar += forward(A, uW) and A_bar += dA(A, uW, dB), with uW folded into a
    // second coefficient table; the kernels add into the outputs (accum)
    Params q2 = q;
    q2.W = uW;
    q2.coef = (float*)((char*)ws + w.coef2);
    q2.coef_r = (float*)((char*)ws + w.coef_r2);
    q2.accum = 1;
    {
      Timed tm(p, K_FOLD, st);
      void* a2[] = {&q2};
      s = cuda_err(cudaLaunchKernel((const void*)p->k_fold, dim3(p->t.E, (p->t.K + 31) / 32, p->kc.fold_split), dim3(128), a2, 0, st),
                   "launch symcon_fold (uW)");
    }
    if (s) return s;
    n++;
    if (dB_bar) {
      q2.B = dB_bar;
      if ((s = launch_fwd_kernel(p, w, q2, N, st))) return s;
      n++;
    }
    if (A_bar) {
      q2.dA = A_bar;
      if ((s = launch_dA_kernel(p, w, q2, st))) return s;
      n++;
    }
  }
  p->last_launches = n;
  return cuda_err(cudaGetLastError(), "backward2 launch");
}

static symcon_status peer_common(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                 int64_t n, uint32_t epoch, uint32_t* epoch_dev, int32_t algo, int64_t spin_limit,
                                 float* out, int32_t* err, void* stream);

symcon_status symcon_peer_allreduce(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                    int64_t n, uint32_t epoch, float* out, int32_t* err, void* stream) {
  return peer_common(bufs, pads, world, rank, n, epoch, nullptr, 1, 0, out, err, stream);
}

symcon_status symcon_peer_allreduce_dev(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                        int64_t n, uint32_t* epoch_counter, float* out, int32_t* err, void* stream) {
  if (!epoch_counter) { set_error("NULL epoch counter"); return SYMCON_EINVAL; }
  return peer_common(bufs, pads, world, rank, n, 0, epoch_counter, 1, 0, out, err, stream);
}

symcon_status symcon_peer_allreduce_ex(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                       int64_t n, uint32_t epoch, uint32_t* epoch_counter, int32_t algo,
                                       int64_t spin_limit, float* out, int32_t* err, void* stream) {
  if (algo < 0 || algo > 2) { set_error("algo must be 0 (auto), 1 (one-shot) or 2 (two-shot)"); return SYMCON_EINVAL; }
  if (spin_limit < 0) { set_error("spin_limit must be >= 0"); return SYMCON_EINVAL; }
  if (algo == 0) algo = world >= 8 ? 2 : 1;   // measured: one-shot faster at 2 and 4
  return peer_common(bufs, pads, world, rank, n, epoch, epoch_counter, algo, spin_limit, out, err, stream);
}

symcon_status symcon_peer_check(const int32_t* err, void* stream) {
  if (!err) { set_error("NULL err"); return SYMCON_EINVAL; }
  symcon_status s = cuda_err(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
  if (s) return s;
  int32_t e = 0;
  s = cuda_err(cudaMemcpy(&e, err, sizeof e, cudaMemcpyDeviceToHost), "read all-reduce error word");
  if (s) return s;
  if (e) { set_error("peer all-reduce barrier timed out: a rank did not arrive (output set to NaN)"); return SYMCON_ETIMEOUT; }
  return SYMCON_OK;
}

static symcon_status peer_common(const float* const* bufs, uint32_t* const* pads, int32_t world, int32_t rank,
                                 int64_t n, uint32_t epoch, uint32_t* epoch_dev, int32_t algo, int64_t spin_limit,
                                 float* out, int32_t* err, void* stream) {
  if (!bufs || !pads || !out || world < 1 || world > 8 || rank < 0 || rank >= world || n < 0) {
    set_error("bad peer all-reduce arguments");
    return SYMCON_EINVAL;
  }
  if (!aligned16(out)) { set_error("out must be 16-byte aligned"); return SYMCON_EINVAL; }
  PeerArgs a{};
  for (int r = 0; r < world; r++) {
    if (!bufs[r] || !pads[r]) { set_error("NULL peer pointer"); return SYMCON_EINVAL; }
    if (!aligned16(bufs[r])) { set_error("peer buffers must be 16-byte aligned"); return SYMCON_EINVAL; }
    a.buf[r] = bufs[r];
    a.pad[r] = pads[r];
  }
  // default ~2^26 polls of ~200 ns: tens of seconds (a rank checkpointing or evaluating must not
  // trip it; a dead rank still ends in a reported error instead of a hang)
  const long long limit = spin_limit > 0 ? (long long)spin_limit : (1ll << 26);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long n4 = (n + 3) / 4;
  a.out[rank] = out;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(sms, (n4 + 511) / 512));
  peer_allreduce_launch(a, world, rank, n, epoch, epoch_dev, algo, limit, err, blocks, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError(), "peer all-reduce launch");
}

symcon_status symcon_peer_allreduce_emulate(const float* const* bufs, uint32_t* const* pads, float* const* outs,
                                            int32_t world, int64_t n, uint32_t epoch, int32_t algo, int64_t spin_limit,
                                            int32_t* err, void* stream) {
  if (!bufs || !pads || !outs || world < 1 || world > 8 || n < 0 || algo < 1 || algo > 2) {
    set_error("bad emulated all-reduce arguments");
    return SYMCON_EINVAL;
  }
  PeerArgs a{};
  for (int r = 0; r < world; r++) {
    if (!bufs[r] || !pads[r] || !outs[r] || !aligned16(bufs[r]) || !aligned16(outs[r])) {
      set_error("NULL or misaligned buffer");
      return SYMCON_EINVAL;
    }
    a.buf[r] = bufs[r];
    a.pad[r] = pads[r];
    a.out[r] = outs[r];
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // all world x blocks CTAs of 512 threads must be co-resident (at most 2 per SM here)
  const long long n4 = (n + 3) / 4;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(std::min(sms, std::max(1, 2 * sms / world)), (n4 + 511) / 512));
  const long long limit = spin_limit > 0 ? (long long)spin_limit : (1ll << 26);
  if (peer_allreduce_launch(a, world, -1, n, epoch, nullptr, algo, limit, err, blocks, (cudaStream_t)stream) < 0)
    return cuda_err(cudaGetLastError(), "cooperative launch of the emulated all-reduce");
  return cuda_err(cudaGetLastError(), "emulated all-reduce launch");
}

symcon_status symcon_check_device_error(const symcon_plan* p, void* ws, void* stream, int64_t* first_bad) {
  if (!p || !ws) { set_error("NULL argument"); return SYMCON_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  symcon_status s = cuda_err(cudaStreamSynchronize(st), "stream sync");
  if (s) return s;
  WsLayout w = layout(p, 0);
  unsigned long long e = 0;
  s = cuda_err(cudaMemcpy(&e, (char*)ws + w.err, sizeof e, cudaMemcpyDeviceToHost), "read error word");
  if (s) return s;
  if (e != ~0ull) {
    if (first_bad) *first_bad = (int64_t)e;
    set_error("node_elem out of range at node " + std::to_string(e));
    return SYMCON_EELEMENT;
  }
  if (first_bad) *first_bad = -1;
  return SYMCON_OK;
}

/* Launch timer: when on, each launch group is bracketed by CUDA events on its stream. */
symcon_status symcon_profile_enable(const symcon_plan* p, int on) {
  if (!p) return SYMCON_EINVAL;
  p->prof_on = on != 0;
  return SYMCON_OK;
}

symcon_status symcon_profile_reset(const symcon_plan* p) {
  if (!p) return SYMCON_EINVAL;
  std::lock_guard<std::mutex> g(p->prof_mu);
  drain(p);
  for (int i = 0; i < SYMCON_PROFILE_MAX; i++) { p->prof_ms[i] = 0; p->prof_n[i] = 0; }
  return SYMCON_OK;
}

/* Synchronises the recorded events; fills up to SYMCON_PROFILE_MAX (name, launches, total ms) entries. */
int32_t symcon_profile_read(const symcon_plan* p, const char** names, int64_t* counts, double* total_ms) {
  if (!p) return 0;
  std::lock_guard<std::mutex> g(p->prof_mu);
  drain(p);
  int n = 0;
  for (int i = 0; i < K_NKINDS; i++)
    if (p->prof_n[i]) {
      if (names) names[n] = kKindNames[i];
      if (counts) counts[n] = p->prof_n[i];
      if (total_ms) total_ms[n] = p->prof_ms[i];
      n++;
    }
  return n;
}

void symcon_destroy(symcon_plan* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> g(p->prof_mu);
    for (auto& r : p->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : p->event_pool) cudaEventDestroy(e);
  }
  if (p->aux) cudaStreamDestroy(p->aux);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->lib) cudaLibraryUnload(p->lib);
  delete p;
}

symcon_status symcon_pack_balanced(const int64_t* sizes, int64_t n, int64_t C, int32_t G, int64_t* bin_offsets,
                                   int64_t* graph_ids, int64_t max_bins, int64_t* n_bins) {
  if (!n_bins || (n > 0 && !sizes) || C < 1 || G < 1 || n < 0) { set_error("bad argument"); return SYMCON_EINVAL; }
  for (int64_t i = 0; i < n; i++)
    if (sizes[i] > C || sizes[i] < 0) { set_error("graph " + std::to_string(i) + " larger than capacity"); return SYMCON_EINVAL; }
  std::vector<std::vector<int64_t>> bins;
  pack_balanced(sizes, n, C, G, bins);
  *n_bins = (int64_t)bins.size();
  if ((int64_t)bins.size() > max_bins || !bin_offsets || (n > 0 && !graph_ids)) { set_error("max_bins too small"); return SYMCON_ENOMEM; }
  int64_t o = 0;
  for (size_t b = 0; b < bins.size(); b++) {
    bin_offsets[b] = o;
    for (int64_t g : bins[b]) graph_ids[o++] = g;
  }
  bin_offsets[bins.size()] = o;
  return SYMCON_OK;
}

}  // extern "C"

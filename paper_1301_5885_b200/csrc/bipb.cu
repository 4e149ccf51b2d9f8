// bipb.cu — the C ABI (include/bipb.h) over the sm_100a kernels: context, device data
// layout, launch configuration, the device-resident GMRES(m) driver and the NCCL
// row-sharded exchange.  Paper: Geng & Jacob, arXiv 1301.5885 (Table 1).
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bipb.h"
#include "bipb_kernels.cuh"
#include "bipb_vec.cuh"
#include "bipb_sym.cuh"
#include "bipb_p2p.cuh"

using namespace bipb;

// ----------------------------------------------------------------- configuration
// One CTA = TPB threads x T targets per thread against one source chunk.
#ifndef BIPB_MV_TPB
#define BIPB_MV_TPB 128
#endif
#ifndef BIPB_MV_T
#define BIPB_MV_T 3
#endif
#ifndef BIPB_MV_MINB
#define BIPB_MV_MINB 3
#endif
constexpr int MV_TPB = BIPB_MV_TPB, MV_T = BIPB_MV_T, MV_MINB = BIPB_MV_MINB;
// symmetric kernel launch shapes per number of right-hand sides R (B = TPB*T rows per block)
#ifndef BIPB_SYM_TPB
#define BIPB_SYM_TPB 128
#endif
#ifndef BIPB_SYM_T
#define BIPB_SYM_T 5
#endif
#ifndef BIPB_SYM_MINB
#define BIPB_SYM_MINB 1
#endif
template <int R>
struct SymCfg;
template <>
struct SymCfg<1> {
  static constexpr int TPB = BIPB_SYM_TPB, T = BIPB_SYM_T, MINB = BIPB_SYM_MINB;
};
#ifndef BIPB_SYM2_T
#define BIPB_SYM2_T 4  // shape sweep at C4 (profiles/r01/tune_batch2_C4.jsonl): R = 2 T = 4 236.9 ms, T = 2 257.3
#endif
#ifndef BIPB_SYM4_T
#define BIPB_SYM4_T 3  // R = 4: T = 3 328.7 ms, T = 2 367.0
#endif
template <>
struct SymCfg<2> {
  static constexpr int TPB = 128, T = BIPB_SYM2_T, MINB = 1;
};
template <>
struct SymCfg<4> {
  static constexpr int TPB = 128, T = BIPB_SYM4_T, MINB = 1;
};
// R = 1 on mid-size problems (fewer than SYM_SMALL_TASKS block pairs at T = 5): smaller blocks,
// 3 CTAs per SM -- more, shorter (I, J) tasks balance better over 148 SMs (measured: C2 product
// 0.966 -> 0.863 ms; C3/C4 are faster at T = 5; profiles/r01/tune_shape_C*.jsonl)
#ifndef BIPB_SYMMID_T
#define BIPB_SYMMID_T 3
#endif
#ifndef BIPB_SYMMID_MINB
#define BIPB_SYMMID_MINB 3
#endif
struct SymCfgMid {
  static constexpr int TPB = 128, T = BIPB_SYMMID_T, MINB = BIPB_SYMMID_MINB;
};
// R = 1 on small problems (fewer than SYM_MID_TASKS block pairs at B = 384, e.g. C1): one target per
// thread, B = 128, 4 CTAs per SM -- enough (I, J) tasks to fill the machine (C1: 840 tasks; product
// 89 us vs 107 us for the row kernel and 153 us at B = 384, profiles/r02/session4/tune_small_C*.jsonl)
struct SymCfgSmall {
  static constexpr int TPB = 128, T = 1, MINB = 4;
};
constexpr int64_t SYM_MID_TASKS = 1024;
constexpr int64_t SYM_MIN_TASKS = 296;  // default kernel: symmetric from this many B = 128 tasks on
static int64_t sym_tasks(int64_t n, int64_t B) {
  const int64_t nb = (n + B - 1) / B;
  return nb * (((nb & 1) ? (nb - 1) / 2 : nb / 2) + 1);
}
constexpr int64_t SYM_SMALL_TASKS = 2048;
static_assert((SymCfg<1>::TPB * SymCfg<1>::T) % TILE == 0, "symmetric block must be a multiple of the smem tile");
static_assert((SymCfgMid::TPB * SymCfgMid::T) % TILE == 0, "symmetric block must be a multiple of the smem tile");
static_assert((SymCfgSmall::TPB * SymCfgSmall::T) % TILE == 0, "symmetric block must be a multiple of the smem tile");
constexpr int SRC_TPB = 128, SRC_T = 2, SRC_MINB = 4;
#ifndef BIPB_EN_T
#define BIPB_EN_T 4  // r02 A/B (profiles/r02/session4/tune_energy_C*.jsonl): C4 3.69 -> 3.40 ms with the wave rule
#endif
#ifndef BIPB_EN_MINB
#define BIPB_EN_MINB 2
#endif
constexpr int EN_TPB = 128, EN_T = BIPB_EN_T, EN_MINB = BIPB_EN_MINB;
constexpr int64_t WANT_CTAS = 148 * 16;  // enough CTAs for a short dynamic-scheduling tail

// NVTX ranges per phase (SURVEY.md §5 "tracing"): visible in nsys / ncu --nvtx timelines; a no-op
// when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;
static bipb_status fail(bipb_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(e_ == cudaErrorMemoryAllocation ? BIPB_ERR_OOM : BIPB_ERR_CUDA,                 \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                            \
  } while (0)
#define CKS(st)                       \
  do {                                \
    bipb_status s_ = (st);            \
    if (s_ != BIPB_OK) return s_;     \
  } while (0)

// ------------------------------------------------------------ NCCL via dlopen
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // failure handling (optional symbols: the one-GPU test stand-in has neither)
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  bool ok = false;
};
static NcclApi load_nccl() {
  NcclApi api;
  // BIPB_NCCL_LIB: explicit library (tests use a one-GPU stand-in, tests/fakenccl); otherwise
  // reuse an already-loaded libnccl (torch's) when there is one
  if (const char* lib = getenv("BIPB_NCCL_LIB")) api.h = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (api.h) break;
    api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
  }
  if (api.h) {
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
    api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
    api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    api.CommAbort = (decltype(api.CommAbort))dlsym(api.h, "ncclCommAbort");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(api.h, "ncclCommGetAsyncError");
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.AllReduce && api.CommDestroy &&
             api.GetErrorString;
  }
  return api;
}
static NcclApi& nccl() {
  static NcclApi api = load_nccl();  // thread-safe one-time initialisation
  return api;
}

// ------------------------------------------------------------------ context
struct EventPool {
  std::vector<cudaEvent_t> ev;  // pairs
  size_t used = 0;
  int64_t launches = 0;
};

struct bipb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  bool sharded = false;  // a bipb_dist was given: stage -> all-gather -> unpack path (even at world 1)
  bool no_comm = false;  // BIPB_DIST_NO_COMM: rows of this rank only (tests)
  ncclComm_t comm = nullptr;

  int64_t n = 0, nc = 0;
  double eps1 = 1, eps2 = 1, kappa = 0, eps = 1, s = 1;
  bool screened = false;
  int64_t r0 = 0, r1 = 0, np = 0;  // element rows of this rank; padded rows per rank
  int64_t k0 = 0, k1 = 0, kp = 0;  // charges of this rank; padded per rank

  // device data
  double *ex = nullptr, *ey = nullptr, *ez = nullptr;     // element centroids x s
  double *enx = nullptr, *eny = nullptr, *enz = nullptr;  // unit normals
  double* ew = nullptr;                                   // areas
  double* rec_el = nullptr;                               // [n][8] source records
  double *qx = nullptr, *qy = nullptr, *qz = nullptr;     // charge positions x s
  double* q4 = nullptr;                                   // [nc][4] raw charges (x,y,z,Q)
  double* rec_ch = nullptr;                               // [nc][4] {x s, y s, z s, Q}
  double* part = nullptr;
  size_t part_cap = 0;
  double* b = nullptr;
  bool have_b = false;
  double* stage = nullptr;   // [2 np] or [kp]
  int64_t stage_cap = 0;
  double* gather = nullptr;  // [world][2 np]
  double *ubuf = nullptr, *ybuf = nullptr, *xbuf = nullptr, *bbuf = nullptr, *tbuf = nullptr;
  double* phit = nullptr;  // [nc]
  double* phi = nullptr;   // [nc]
  // GMRES
  double* V = nullptr;
  int m_cap = 0;
  double *H = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr, *yk = nullptr;
  double* scal = nullptr;  // scalars: [0] beta_b^2, [1] beta, [2] hk1sq, [3] hk1, [4] tmp, [5] energy, [6..7] info
  double* red_part = nullptr;
  unsigned* red_cnt = nullptr;
  double* host_info = nullptr;  // pinned [4]
  double* host_info_dev = nullptr;  // its device mapping (UVA), or null
  int arn_E = -1;                   // fused Arnoldi tail: elements per thread (0 = multi-launch MGS)
  int precond = 0;                  // 0 plain GMRES (paper), 1 right jump-term diagonal (bipb_set_precond)
  double pinv1 = 1.0, pinv2 = 1.0;  // M^-1 on the phi / dphi rows
  double* zbuf = nullptr;           // M^-1 v_k (2n)
  int* dflag = nullptr;

  // symmetric matvec (bipb_sym.cuh): one schedule per R in {1, 2, 4}
  int mv_kind = 1;  // 0 = row kernel (one evaluation per ordered pair), 1 = symmetric
  struct SymPlan {
    int R = 0;
    int64_t B = 0, nb = 0, hmax = 0, W = 1, runs = 1, I0 = 0, I1 = 0, group = 1;
    double *rec = nullptr, *fwd = nullptr, *rev = nullptr;
  } sym[3];
  double* sym_P = nullptr;  // [4][2][n] running row sums
  // exact sums of the single-operand symmetric product (bipb_exact.cuh; bipb_set_sum_mode)
  int sum_mode = 1;                   // 1 exact fixed-point limbs (default), 0 fixed-order double partials
  bool exact_off = false;             // set after an out-of-range partial: double partials from then on
  unsigned long long* xl = nullptr;   // [3][2n] row limbs + overflow count
  int* xexp = nullptr;                // operand exponent max
  int* xsticky = nullptr;             // set by finish_exact_kernel when a product overflowed
  int xbias = 0;                      // BIPB_EXACT_BIAS test hook
  double* x0save = nullptr;           // GMRES x0 kept for the double-partial rerun
  double* bat_U = nullptr;  // [4][2n] batch staging (host inputs)
  double* bat_Y = nullptr;
  int64_t chunk_mv = 0, nchunk_mv = 0, chunk_src = 0, nchunk_src = 0, chunk_en = 0, nchunk_en = 0;
  int64_t en_resident = 0;  // SMs x resident energy-kernel CTAs per SM (whole-wave chunk rule)
  // peer-store exchange of the products (bipb_p2p.cuh; BIPB_DIST_P2P / BIPB_EXCHANGE=p2p)
  bool p2p = false;
  double* p2p_box = nullptr;                // own mailbox [2][stride] (cudaMalloc: IPC-exportable)
  unsigned long long* p2p_flags = nullptr;  // own flags [world] (written by the peers)
  unsigned long long* p2p_epoch = nullptr;  // own exchange counter (device)
  int64_t p2p_stride = 0;
  PeerBoxes boxes{};
  PeerFlags flags{};
  std::vector<void*> p2p_opened;  // peer mappings to close
  unsigned long long p2p_timeout_ns = 120ull * 1000000000ull;  // peer-store delivery (BIPB_P2P_TIMEOUT_S)
  unsigned long long comm_timeout_ns = 600ull * 1000000000ull; // host watchdog (BIPB_COMM_TIMEOUT_S)
  unsigned int* p2p_err = nullptr;      // mapped pinned word: 1 + rank that missed a delivery (p2p_wait_kernel)
  unsigned int* p2p_err_dev = nullptr;  // its device address
  // a peer that missed a delivery or a failed / stuck collective leaves the context unusable: every
  // later call returns BIPB_ERR_NCCL with this message (destroy the context)
  bool failed = false;
  std::string failed_msg;

  bool timing = false;
  EventPool pool[3];
  int64_t launches_all = 0;
  int64_t matvec_calls = 0;  // operator applications (for per-product kernel time)
  int warm_kind = -1;        // 2 kind + exact sums: the product whose buffers / attributes exist (eager product done)
  // CUDA graphs of the GMRES Arnoldi steps (one per k), valid for (V, m, n, kind)
  struct {
    const double* V = nullptr;
    int m = 0, kind = -1, precond = -1, exact = -1;
    std::vector<cudaGraphExec_t> ex;
  } ag;
  // BIPB_GRAPHS=2: one graph per Arnoldi cycle (m IF nodes, each one step + cycle_check_kernel),
  // same validity key as `ag`; cyc = device [8 + 2m] (parameters, per-step records), cyc_host its
  // pinned copy
  struct {
    const double* V = nullptr;
    int m = 0, kind = -1, precond = -1, exact = -1;
    cudaGraphExec_t ex = nullptr;
  } cg;
  double* cyc = nullptr;
  double* cyc_host = nullptr;
  int cyc_cap = 0;
  int64_t graph_cycles = 0;  // cycles run as one graph launch (bipb_get_graph_cycles)
  bool cycle_off = false;  // the cycle graph could not be built here: eager cycles from then on
  std::string cycle_err;
};

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// BIPB_TRACE=1: host wall-clock phases of bipb_setup on stderr (tools/e2e_breakdown.py)
struct Trace {
  bool on = getenv("BIPB_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[bipb] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

// Source chunk length for a pair launch: chosen from GLOBAL sizes only, so a row's sum
// order (and value) does not depend on the number of ranks.
static int64_t choose_chunk(int64_t ntgt_global, int64_t nsrc, int tgt_per_cta) {
  const int64_t tiles = std::max<int64_t>(1, cdiv(ntgt_global, tgt_per_cta));
  int64_t nchunk = std::max<int64_t>(32, cdiv(WANT_CTAS, tiles));
  nchunk = std::min<int64_t>(nchunk, std::max<int64_t>(1, cdiv(nsrc, TILE)));
  int64_t chunk = cdiv(cdiv(nsrc, nchunk), TILE) * TILE;
  return std::max<int64_t>(chunk, TILE);
}

// Energy launch (few charge tiles x many element chunks): the chunk count is
// rounded so that tiles x chunks fills whole waves of `resident` CTAs (r01 ncu: 2,340 CTAs over
// 888 resident slots = 2.64 waves, FP64 pipe 77%).  Chunks stay >= one smem tile; below one wave
// the rule is choose_chunk's.  `resident` is a device property (SMs x occupancy), equal on every
// rank, so the sum order stays independent of the rank count.  BIPB_EN_WAVES=0 disables it (A/B).
static int64_t choose_chunk_waves(int64_t ntgt_global, int64_t nsrc, int tgt_per_cta, int64_t resident) {
  static const bool on = !(getenv("BIPB_EN_WAVES") && !strcmp(getenv("BIPB_EN_WAVES"), "0"));
  if (!on || resident <= 0) return choose_chunk(ntgt_global, nsrc, tgt_per_cta);
  const int64_t tiles = std::max<int64_t>(1, cdiv(ntgt_global, tgt_per_cta));
  const int64_t cap = std::max<int64_t>(1, cdiv(nsrc, TILE));
  int64_t want = std::min<int64_t>(std::max<int64_t>(32, cdiv(WANT_CTAS, tiles)), cap);
  if (tiles * want >= resident) {
    const int64_t waves = cdiv(tiles * want, resident);
    want = std::min<int64_t>(cap, std::max<int64_t>(1, waves * resident / tiles));
  }
  return std::max<int64_t>(1, cdiv(nsrc, want));
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Where a vector argument lives: host memory (pageable or pinned) -> *dev = false; device or
// managed memory of the context's GPU -> *dev = true; another GPU's memory -> ERR_ARG (the
// kernels would read it through peer mappings that may not exist).
static bipb_status vec_where(bipb_ctx* c, const void* p, bool* dev);

static void launch_1d_cfg(int64_t work, int& grid, int& block) {
  block = 256;
  grid = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(work, block)), 148 * 8);
}

static bipb_status timed_begin(bipb_ctx* c, int which, cudaEvent_t* stop_out) {
  *stop_out = nullptr;
  c->pool[which].launches++;
  c->launches_all++;
  if (!c->timing) return BIPB_OK;
  EventPool& p = c->pool[which];
  if (p.used + 2 > p.ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      p.ev.push_back(e);
    }
  }
  CK(cudaEventRecord(p.ev[p.used], c->stream));
  *stop_out = p.ev[p.used + 1];
  p.used += 2;
  return BIPB_OK;
}

// opt-in dynamic shared memory, set once per (device, kernel, size) (the attribute call costs
// tens of microseconds; GMRES on small meshes launches a pair kernel every iteration)
template <typename KernelT>
static bipb_status set_smem(KernelT k, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const auto key = std::make_pair(dev, reinterpret_cast<const void*>(k));
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return BIPB_OK;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  done[key] = smem;
  return BIPB_OK;
}

// pair launches ----------------------------------------------------------------
template <int MODE, int TPB, int T, int MINB>
static bipb_status launch_pair(bipb_ctx* c, const PairArgs& a, int64_t nchunk, int which) {
  if (a.ntgt <= 0) return BIPB_OK;
  constexpr int REC = (MODE == SOURCE) ? 4 : 8;
  const size_t smem = sizeof(double) * STAGES * TILE * REC + 8 * STAGES;
  dim3 grid((unsigned)cdiv(a.ntgt, TPB * T), (unsigned)nchunk);
  if (grid.y > 65535) return fail(BIPB_ERR_ARG, "too many source chunks");
  cudaEvent_t stop;
  CKS(timed_begin(c, which, &stop));
  if (c->screened) {
    auto k = pair_kernel<MODE, TPB, T, true, MINB>;
    CKS(set_smem(k, smem));
    k<<<grid, TPB, smem, c->stream>>>(a);
  } else {
    auto k = pair_kernel<MODE, TPB, T, false, MINB>;
    CKS(set_smem(k, smem));
    k<<<grid, TPB, smem, c->stream>>>(a);
  }
  CK(cudaGetLastError());
  if (stop) CK(cudaEventRecord(stop, c->stream));
  return BIPB_OK;
}

// Device memory comes from the device's default stream-ordered pool, configured to retain freed
// memory (release threshold = max): contexts created and destroyed per solve (the e2e path)
// then neither pay cudaMalloc nor the occasional multi-100-ms cudaFree trim of large blocks.
static void pool_init_once(int dev) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done.push_back(dev);
}
template <typename T>
static cudaError_t dmalloc(bipb_ctx* c, T** p, size_t bytes) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, c->stream);
}
static void dfree(bipb_ctx* c, void* p) {
  if (p) cudaFreeAsync(p, c->stream);
}

static void drop_graphs(bipb_ctx* c) {
  if (c->stream) cudaStreamSynchronize(c->stream);  // no replay of them is still pending
  for (auto e : c->ag.ex)
    if (e) cudaGraphExecDestroy(e);
  c->ag.ex.clear();
  c->ag.V = nullptr;  // forces a rebuild on the next solve
  if (c->cg.ex) cudaGraphExecDestroy(c->cg.ex);
  c->cg.ex = nullptr;
  c->cg.V = nullptr;
}

// chunk-partial scratch of the row kernel / source / energy, grown on demand.  A reallocation
// invalidates the cached Arnoldi-step graphs, which bake the old pointer into their row-kernel
// products (a replay would otherwise write into freed pool memory).
static bipb_status ensure_part(bipb_ctx* c, size_t doubles) {
  if (doubles <= c->part_cap) return BIPB_OK;
  if (c->part) {
    drop_graphs(c);
    dfree(c, c->part);
  }
  c->part = nullptr;
  CK(dmalloc(c, &c->part, doubles * sizeof(double)));
  c->part_cap = doubles;
  return BIPB_OK;
}

#define LAUNCH1D(kern, work, ...)                                   \
  do {                                                              \
    int g_, b_;                                                     \
    launch_1d_cfg((work), g_, b_);                             \
    kern<<<g_, b_, 0, c->stream>>>(__VA_ARGS__);                    \
    c->launches_all++;                                              \
    CK(cudaGetLastError());                                         \
  } while (0)

static void p2p_teardown(bipb_ctx* c) {
  cudaStreamSynchronize(c->stream);
  for (void* q : c->p2p_opened) cudaIpcCloseMemHandle(q);
  c->p2p_opened.clear();
  if (c->p2p_box) cudaFree(c->p2p_box);
  if (c->p2p_flags) cudaFree(c->p2p_flags);
  c->p2p_box = nullptr;
  c->p2p_flags = nullptr;
  c->boxes = PeerBoxes{};
  c->flags = PeerFlags{};
  cudaGetLastError();
}


// ---- failure handling of the multi-GPU exchange (SURVEY.md §5 "failure detection")
// Marks the context failed; aborts the communicator so NCCL kernels still waiting on a peer exit.
static bipb_status ctx_fail(bipb_ctx* c, const std::string& msg) {
  if (!c->failed) {
    c->failed = true;
    c->failed_msg = msg;
    if (c->comm && nccl().CommAbort) {
      nccl().CommAbort(c->comm);
      c->comm = nullptr;
    }
  }
  return fail(BIPB_ERR_NCCL, msg);
}
static bipb_status nccl_check(bipb_ctx* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return BIPB_OK;
  return ctx_fail(c, std::string(what) + ": " + nccl().GetErrorString(r));
}
static bipb_status check_alive(bipb_ctx* c) {
  if (c->failed) return fail(BIPB_ERR_NCCL, "context failed earlier (" + c->failed_msg + "); destroy it");
  return BIPB_OK;
}
static bipb_status p2p_check(bipb_ctx* c) {
  if (c->p2p && c->p2p_err && *reinterpret_cast<volatile unsigned int*>(c->p2p_err) != 0u)
    return ctx_fail(c, "peer-store exchange: rank " + std::to_string(*c->p2p_err - 1) + " did not deliver within " +
                           std::to_string(c->p2p_timeout_ns / 1000000000ull) + " s (BIPB_P2P_TIMEOUT_S)");
  return BIPB_OK;
}
// Wait for the context's stream.  Single-GPU contexts block in cudaStreamSynchronize.  Sharded
// contexts poll: an NCCL asynchronous error, or stream work still running after the host watchdog
// (BIPB_COMM_TIMEOUT_S, default 600 s per synchronisation -- far above one product: C5 on one GPU
// takes 8.6 s) aborts the communicator and returns BIPB_ERR_NCCL instead of hanging; a missed
// peer-store delivery is reported from the wait kernel's error word.
static bipb_status ctx_sync(bipb_ctx* c) {
  if (!c->sharded || c->no_comm) {
    CK(cudaStreamSynchronize(c->stream));
    return BIPB_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  for (;;) {
    const cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) CK(e);
    if (c->comm && nccl().CommGetAsyncError) {
      ncclResult_t ar = ncclSuccess;
      if (nccl().CommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
        return ctx_fail(c, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ar));
    }
    const auto el = std::chrono::steady_clock::now() - t0;
    if ((unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(el).count() > c->comm_timeout_ns)
      return ctx_fail(c, "exchange did not complete within BIPB_COMM_TIMEOUT_S (" +
                             std::to_string(c->comm_timeout_ns / 1000000000ull) + " s)");
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  return p2p_check(c);
}

// exchange: every rank's rows [r0,r1) of the two halves -> full vector on every rank
static bipb_status allgather_rows(bipb_ctx* c, double* y) {
  if (c->no_comm) {  // test mode: place this rank's rows only
    CK(cudaMemsetAsync(y, 0, 2 * c->n * sizeof(double), c->stream));
    CK(cudaMemsetAsync(c->gather, 0, (size_t)c->world * 2 * c->np * sizeof(double), c->stream));
    CK(cudaMemcpyAsync(c->gather + (size_t)c->rank * 2 * c->np, c->stage, 2 * c->np * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->stream));
    LAUNCH1D(unpack_kernel, c->world * c->np, c->gather, c->n, c->np, c->world, y);
    return BIPB_OK;
  }
  NcclApi& api = nccl();
  CKS(nccl_check(c, api.AllGather(c->stage, c->gather, (size_t)(2 * c->np), ncclFloat64, c->comm, c->stream),
                 "ncclAllGather"));
  LAUNCH1D(unpack_kernel, c->world * c->np, c->gather, c->n, c->np, c->world, y);
  return BIPB_OK;
}

// ---- peer-store exchange (bipb_p2p.cuh): the producer kernel already stored its values into
// every rank's mailbox; publish the epoch and wait for every rank's delivery.
static bipb_status p2p_publish_and_wait(bipb_ctx* c) {
  p2p_signal_kernel<<<1, 32, 0, c->stream>>>(c->p2p_epoch, c->flags, c->world, c->rank);
  p2p_wait_kernel<<<1, 32, 0, c->stream>>>(c->p2p_epoch, c->p2p_flags, c->world, c->p2p_timeout_ns,
                                            c->p2p_err_dev);
  c->launches_all += 2;
  CK(cudaGetLastError());
  return BIPB_OK;
}

// ---- symmetric-pair products (bipb_sym.cuh) ------------------------------------------------
static int sym_slot(int R) { return R == 1 ? 0 : (R == 2 ? 1 : 2); }

// Per-R schedule (global sizes; this rank's I-blocks) and buffers, allocated on first use.
// Partials are bounded by BIPB_SYM_MEM_GB (default 4) by launching the rank's I-blocks in groups.
template <int R>
static bipb_status sym_plan(bipb_ctx* c, bipb_ctx::SymPlan** out) {
  bipb_ctx::SymPlan& p = c->sym[sym_slot(R)];
  *out = &p;
  if (p.R == R) return BIPB_OK;
  constexpr int F = SymLayout<R>::F;
  const int64_t n = c->n;
  int64_t B = SymCfg<R>::TPB * SymCfg<R>::T;
  if (R == 1 && sym_tasks(n, B) < SYM_SMALL_TASKS) {  // fewer, larger tasks than the machine wants
    B = SymCfgMid::TPB * SymCfgMid::T;
    if (sym_tasks(n, B) < SYM_MID_TASKS) B = SymCfgSmall::TPB * SymCfgSmall::T;
  }
  p.B = B;
  p.nb = cdiv(n, B);
  p.hmax = (p.nb & 1) ? (p.nb - 1) / 2 : p.nb / 2;
  bipb_partition(p.nb, c->world, c->rank, &p.I0, &p.I1);
  // runs of W offsets per CTA, chosen from GLOBAL sizes only: a run's forward sums form one partial,
  // so a W that depended on the rank's share (as in r01: >= 32 waves per rank) would group the
  // partials differently on P ranks and the exact-sum product would differ from the single-GPU one
  // in the last bits at large N (r02 session 4: the 8-rank C4 product).  W = 2 from 16 waves of
  // 2 CTAs/SM per rank at 8 ranks (37,888 block pairs) on, else 1: short CTAs of nearly equal work
  // keep the tail small on 1-8 GPUs (C4 per product: W = 1 192.5 ms, 2 191.4, 4 191.6; r01 W sweep
  // 16 192.7, 8 192.8, 6 191.9 -- profiles/r02/session4/tune_fpo_C4.jsonl, r01/session3/sweepW_C4.jsonl)
  const int64_t tiles_global = p.nb * (p.hmax + 1);
  p.W = tiles_global >= (int64_t)8 * 148 * 2 * 16 ? 2 : 1;
  if (const char* e = getenv("BIPB_SYM_W")) p.W = std::max<int64_t>(1, atoll(e));  // tuning
  p.runs = cdiv(p.hmax + 1, p.W);  // an I-block's offsets split evenly over its runs (bipb_sym.cuh)
  double gb = 4.0;
  if (const char* e = getenv("BIPB_SYM_MEM_GB")) gb = std::max(0.001, atof(e));
  const double per_block = (double)((p.hmax + 1) + p.runs) * R * 2 * B * sizeof(double);
  p.group = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(p.I1 - p.I0, 1), (int64_t)(gb * 1e9 / per_block)));
  const size_t rec_doubles = (size_t)cdiv(n, TILE) * TILE * F;  // tile-SoA, padded to whole tiles
  CK(dmalloc(c, &p.rec, rec_doubles * sizeof(double)));
  CK(cudaMemsetAsync(p.rec, 0, rec_doubles * sizeof(double), c->stream));
  if (!c->sym_P) CK(dmalloc(c, &c->sym_P, (size_t)4 * 2 * n * sizeof(double)));
  p.R = R;
  return BIPB_OK;
}

// the double partials of a plan, allocated on the first fixed-order product (exact sums need none)
static bipb_status sym_partials(bipb_ctx* c, bipb_ctx::SymPlan* p, int R) {
  if (p->fwd) return BIPB_OK;
  CK(dmalloc(c, &p->fwd, (size_t)p->group * p->runs * R * 2 * p->B * sizeof(double)));
  CK(dmalloc(c, &p->rev, (size_t)p->group * (p->hmax + 1) * R * 2 * p->B * sizeof(double)));
  return BIPB_OK;
}

static bool exact_active(const bipb_ctx* c) { return c->sum_mode == 1 && !c->exact_off && c->mv_kind == 1; }
// which product variant an eager call has prepared (buffers allocated, attributes set): graph
// capture of the Arnoldi steps waits for it
static int warm_key(const bipb_ctx* c) { return 2 * c->mv_kind + (exact_active(c) ? 1 : 0); }

// did an exact product since the last check have an out-of-range partial?  (the flag is derived
// from the exchanged limbs, so every rank sees the same answer)  Switches the context to double
// partials when it did.
static bipb_status exact_overflowed(bipb_ctx* c, bool* out) {
  *out = false;
  if (!c->xsticky) return BIPB_OK;
  int h = 0;
  CK(cudaMemcpyAsync(&h, c->xsticky, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CKS(ctx_sync(c));
  if (h) {
    CK(cudaMemsetAsync(c->xsticky, 0, sizeof(int), c->stream));
    c->exact_off = true;
    *out = true;
  }
  return BIPB_OK;
}

// Y[r] = A U[r] for r < R (device, [R][2n] each; Y must not alias U).  exact: R = 1 with exact
// sums (bipb_exact.cuh) when the context asks for them.
template <int R>
static bipb_status matvec_sym_R(bipb_ctx* c, const double* U, double* Y, bool allow_exact = false) {
  using Cfg = SymCfg<R>;
  const int64_t n = c->n;
  bipb_ctx::SymPlan* p;
  CKS(sym_plan<R>(c, &p));
  const bool exact = R == 1 && allow_exact && exact_active(c);
  const int64_t xwords = 6 * n + 1;
  if (exact) {
    if (!c->xl) {
      CK(dmalloc(c, &c->xl, (size_t)xwords * sizeof(unsigned long long)));
      CK(dmalloc(c, &c->xexp, sizeof(int)));
      CK(dmalloc(c, &c->xsticky, sizeof(int)));
      CK(cudaMemsetAsync(c->xsticky, 0, sizeof(int), c->stream));
    }
    CK(cudaMemsetAsync(c->xl, 0, (size_t)xwords * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->xexp, 0, sizeof(int), c->stream));
  } else {
    CKS(sym_partials(c, p, R));
  }
  LAUNCH1D(prescale_sym_kernel<R>, n, U, c->ew, c->ex, c->ey, c->ez, c->enx, c->eny, c->enz, p->rec, n, c->s,
           exact ? c->xexp : nullptr);
  SymArgs a{};
  a.rec = p->rec; a.n = n; a.nb = p->nb; a.B = p->B; a.runs = p->runs; a.W = p->W; a.hmax = p->hmax;
  a.eps = c->eps; a.inveps = 1.0 / c->eps;
  a.sc1 = c->s; a.sc2 = c->s * c->s;
  a.fwd = p->fwd; a.rev = p->rev;
  a.xl = exact ? c->xl : nullptr; a.xexp = c->xexp; a.xbias = c->xbias;
  const size_t smem =
      sizeof(double) * (STAGES * TILE * SymLayout<R>::F + (Cfg::TPB / 32) * R * 2 * sym_rs_rows(R, (int)p->B)) +
      8 * STAGES;
  const PeerBoxes nobox{};
  if (p->I1 <= p->I0 && !exact) {  // no I-blocks on this rank: its partial sums are zero
    if (c->p2p) {
      LAUNCH1D(reduce_sym_kernel<R>, n, p->fwd, p->rev, n, p->nb, p->B, p->runs, p->hmax, p->I0, p->I0, 1, c->sym_P,
               c->boxes, c->world, c->rank, c->p2p_stride, c->p2p_epoch);
    } else {
      CK(cudaMemsetAsync(c->sym_P, 0, (size_t)R * 2 * n * sizeof(double), c->stream));
    }
  }
  // exact sums need no partial memory: one launch unless BIPB_SYM_MEM_GB asks for groups (tests)
  const int64_t group = (exact && !getenv("BIPB_SYM_MEM_GB")) ? std::max<int64_t>(1, p->I1 - p->I0) : p->group;
  for (int64_t Ia = p->I0; Ia < p->I1; Ia += group) {
    const int64_t Ib = std::min(Ia + group, p->I1);
    a.I0 = Ia;
    const int64_t grid = (Ib - Ia) * p->runs;
    if (grid > 2147483647LL) return fail(BIPB_ERR_ARG, "symmetric grid too large");
    cudaEvent_t stop;
    CKS(timed_begin(c, 0, &stop));
    bool mid = false;
    if constexpr (R == 1) {
      // the smaller R = 1 block shapes (mid-size and small problems)
      auto launch_shape = [&](auto shape) -> bipb_status {
        using M = decltype(shape);
        auto k = c->screened ? (exact ? sym_kernel<M::TPB, M::T, true, M::MINB, R, R == 1>
                                      : sym_kernel<M::TPB, M::T, true, M::MINB, R>)
                             : (exact ? sym_kernel<M::TPB, M::T, false, M::MINB, R, R == 1>
                                      : sym_kernel<M::TPB, M::T, false, M::MINB, R>);
        CKS(set_smem(k, smem));
        k<<<(unsigned)grid, M::TPB, smem, c->stream>>>(a);
        return BIPB_OK;
      };
      if (p->B == SymCfgMid::TPB * SymCfgMid::T) {
        CKS(launch_shape(SymCfgMid{}));
        mid = true;
      } else if (p->B == SymCfgSmall::TPB * SymCfgSmall::T) {
        CKS(launch_shape(SymCfgSmall{}));
        mid = true;
      }
    }
    if (mid) {
    } else if (c->screened) {
      auto k = exact ? sym_kernel<Cfg::TPB, Cfg::T, true, Cfg::MINB, R, R == 1> : sym_kernel<Cfg::TPB, Cfg::T, true, Cfg::MINB, R>;
      CKS(set_smem(k, smem));
      k<<<(unsigned)grid, Cfg::TPB, smem, c->stream>>>(a);
    } else {
      auto k = exact ? sym_kernel<Cfg::TPB, Cfg::T, false, Cfg::MINB, R, R == 1> : sym_kernel<Cfg::TPB, Cfg::T, false, Cfg::MINB, R>;
      CKS(set_smem(k, smem));
      k<<<(unsigned)grid, Cfg::TPB, smem, c->stream>>>(a);
    }
    CK(cudaGetLastError());
    if (stop) CK(cudaEventRecord(stop, c->stream));
    if (exact) continue;
    // the last group's epilogue stores the rank's row sums straight into every rank's mailbox
    const bool to_peers = c->p2p && Ib == p->I1;
    LAUNCH1D(reduce_sym_kernel<R>, n, p->fwd, p->rev, n, p->nb, p->B, p->runs, p->hmax, Ia, Ib, Ia == p->I0 ? 1 : 0,
             c->sym_P, to_peers ? c->boxes : nobox, to_peers ? c->world : 0, c->rank, c->p2p_stride,
             c->p2p_epoch);
  }
  const double d1 = 0.5 * (1.0 + c->eps), d2 = 0.5 * (1.0 + 1.0 / c->eps);
  if (exact) {
    if (c->p2p) {  // limbs into slot [rank] of every mailbox, then the integer sum over the slots
      LAUNCH1D(exact_publish_p2p_kernel, xwords, c->xl, xwords, c->boxes, c->world, c->rank, c->p2p_stride,
               c->p2p_epoch);
      CKS(p2p_publish_and_wait(c));
      LAUNCH1D(finish_exact_kernel, 2 * n, reinterpret_cast<const unsigned long long*>(c->p2p_box), c->p2p_stride,
               c->p2p_epoch, c->world, xwords, c->xexp, c->xbias, U, n, d1, d2, Y, c->xsticky);
    } else {
      if (c->sharded && !c->no_comm) {  // integer sums: exact in any reduction order
        CKS(nccl_check(c, nccl().AllReduce(c->xl, c->xl, (size_t)xwords, ncclUint64, ncclSum, c->comm, c->stream),
                       "ncclAllReduce"));
      }
      LAUNCH1D(finish_exact_kernel, 2 * n, c->xl, 0, nullptr, 1, xwords, c->xexp, c->xbias, U, n, d1, d2, Y,
               c->xsticky);
    }
    c->matvec_calls += 1;
    return BIPB_OK;
  }
  if (c->p2p) {
    CKS(p2p_publish_and_wait(c));
    LAUNCH1D(finish_sym_p2p_kernel<R>, n, c->p2p_box, c->p2p_stride, c->p2p_epoch, c->world, U, n, d1, d2, Y);
    c->matvec_calls += R;
    return BIPB_OK;
  }
  if (c->sharded && !c->no_comm) {  // every rank holds partial sums for all rows
    CKS(nccl_check(c, nccl().AllReduce(c->sym_P, c->sym_P, (size_t)(R * 2 * n), ncclFloat64, ncclSum, c->comm,
                                       c->stream),
                   "ncclAllReduce"));
  }
  LAUNCH1D(finish_sym_kernel<R>, n, c->sym_P, U, n, d1, d2, Y);
  c->matvec_calls += R;
  return BIPB_OK;
}

static bipb_status matvec_sym_dev(bipb_ctx* c, const double* u, double* y) { return matvec_sym_R<1>(c, u, y, true); }

// y = A u (device vectors of length 2n; y must not alias u)
static bipb_status matvec_dev_impl(bipb_ctx* c, const double* u, double* y);
static bipb_status matvec_dev(bipb_ctx* c, const double* u, double* y) {
  CKS(matvec_dev_impl(c, u, y));
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs == cudaStreamCaptureStatusNone) c->warm_kind = warm_key(c);
  return BIPB_OK;
}
static bipb_status matvec_dev_impl(bipb_ctx* c, const double* u, double* y) {
  if (c->mv_kind == 1) return matvec_sym_dev(c, u, y);
  const int64_t n = c->n;
  LAUNCH1D(prescale_kernel, n, u, c->ew, c->enx, c->eny, c->enz, c->rec_el, n);
  const int64_t nloc = c->r1 - c->r0;
  PairArgs a{};
  a.tx = c->ex + c->r0; a.ty = c->ey + c->r0; a.tz = c->ez + c->r0;
  a.tnx = c->enx + c->r0; a.tny = c->eny + c->r0; a.tnz = c->enz + c->r0;
  a.tgt_begin = c->r0; a.ntgt = nloc;
  a.src = c->rec_el; a.nsrc = n; a.chunk = c->chunk_mv;
  a.eps = c->eps; a.inveps = 1.0 / c->eps;
  a.sc1 = c->s; a.sc2 = c->s * c->s; a.sc3 = c->s * c->s * c->s;
  a.part = c->part;
  CKS(ensure_part(c, (size_t)(2 * c->nchunk_mv * std::max<int64_t>(nloc, 1))));
  a.part = c->part;
  CKS((launch_pair<MATVEC, MV_TPB, MV_T, MV_MINB>(c, a, c->nchunk_mv, 0)));
  c->matvec_calls += 1;
  const double d1 = 0.5 * (1.0 + c->eps), d2 = 0.5 * (1.0 + 1.0 / c->eps);
  if (!c->sharded) {
    LAUNCH1D(reduce_matvec_kernel, nloc, c->part, c->nchunk_mv, nloc, u, u + n, d1, d2, y, y + n);
  } else if (c->p2p) {  // epilogue stores the rank's rows into every rank's mailbox
    LAUNCH1D(reduce_matvec_p2p_kernel, std::max<int64_t>(nloc, 1), c->part, c->nchunk_mv, nloc, u + c->r0,
             u + n + c->r0, d1, d2, c->r0, n, c->boxes, c->world, c->p2p_stride, c->p2p_epoch);
    CKS(p2p_publish_and_wait(c));
    LAUNCH1D(p2p_take_kernel, 2 * n, c->p2p_box, c->p2p_stride, c->p2p_epoch, 2 * n, y);
  } else {
    LAUNCH1D(reduce_matvec_kernel, nloc, c->part, c->nchunk_mv, nloc, u + c->r0, u + n + c->r0, d1, d2, c->stage,
             c->stage + c->np);
    CKS(allgather_rows(c, y));
  }
  return BIPB_OK;
}

// ||v||^2 or <a,b> into *out (device)
static bipb_status dot_dev(bipb_ctx* c, const double* a, const double* b, int64_t m, double scale, double* out) {
  dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(a, b, m, scale, c->red_part, c->red_cnt, out);
  c->launches_all++;
  CK(cudaGetLastError());
  return BIPB_OK;
}

static bipb_status read_scalars(bipb_ctx* c, const double* dsrc, int count, double* host) {
  CK(cudaMemcpyAsync(c->host_info, dsrc, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  CKS(ctx_sync(c));
  memcpy(host, c->host_info, sizeof(double) * count);
  return BIPB_OK;
}

static bipb_status vec_where(bipb_ctx* c, const void* p, bool* dev) {
  *dev = false;
  if (!p) return BIPB_OK;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return BIPB_OK;
  }
  if (at.type == cudaMemoryTypeDevice && at.device != c->device)
    return fail(BIPB_ERR_ARG, "vector lives on GPU " + std::to_string(at.device) + ", the context on GPU " +
                                  std::to_string(c->device));
  *dev = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  return BIPB_OK;
}

// input vector -> device pointer (copying host data into `scratch`)
static bipb_status in_vec(bipb_ctx* c, const double* p, int64_t len, double* scratch, const double** out) {
  bool dev;
  CKS(vec_where(c, p, &dev));
  if (dev) {
    *out = p;
    return BIPB_OK;
  }
  CK(cudaMemcpyAsync(scratch, p, sizeof(double) * len, cudaMemcpyHostToDevice, c->stream));
  *out = scratch;
  return BIPB_OK;
}

// ===================================================================== C ABI
extern "C" {

const char* bipb_last_error(void) { return g_err.c_str(); }

const char* bipb_version(void) { return "bipb 0.1 (sm_100a, FP64 direct sum, arXiv 1301.5885)"; }

void bipb_partition(int64_t n, int32_t world, int32_t rank, int64_t* r0, int64_t* r1) {
  if (world < 1) world = 1;
  const int64_t np = cdiv(std::max<int64_t>(n, 0), world);
  int64_t a = std::min<int64_t>((int64_t)rank * np, std::max<int64_t>(n, 0));
  int64_t b = std::min<int64_t>(a + np, std::max<int64_t>(n, 0));
  if (r0) *r0 = a;
  if (r1) *r1 = b;
}

bipb_status bipb_nccl_unique_id(unsigned char* out) {
  if (!out) return fail(BIPB_ERR_ARG, "out is NULL");
  NcclApi& api = nccl();
  if (!api.ok) return fail(BIPB_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(BIPB_ERR_NCCL, api.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return BIPB_OK;
}

void bipb_destroy(bipb_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  double* bufs[] = {c->ex, c->ey, c->ez, c->enx, c->eny, c->enz, c->ew, c->rec_el, c->qx, c->qy, c->qz, c->q4,
                    c->rec_ch, c->part, c->b, c->stage, c->gather, c->ubuf, c->ybuf, c->xbuf, c->bbuf, c->tbuf,
                    c->phit, c->phi, c->V, c->H, c->cs, c->sn, c->g, c->yk, c->scal, c->red_part,
                    c->sym_P, c->bat_U, c->bat_Y, c->zbuf, c->x0save};
  for (double* p : bufs)
    if (p) dfree(c, p);
  for (auto& sp : c->sym) {
    if (sp.rec) dfree(c, sp.rec);
    if (sp.fwd) dfree(c, sp.fwd);
    if (sp.rev) dfree(c, sp.rev);
  }
  if (c->red_cnt) dfree(c, c->red_cnt);
  if (c->dflag) dfree(c, c->dflag);
  if (c->xl) dfree(c, c->xl);
  if (c->xexp) dfree(c, c->xexp);
  if (c->xsticky) dfree(c, c->xsticky);
  if (c->p2p_epoch) dfree(c, c->p2p_epoch);
  if (c->stream) cudaStreamSynchronize(c->stream);
  p2p_teardown(c);
  if (c->p2p_err) cudaFreeHost(c->p2p_err);
  if (c->host_info) cudaFreeHost(c->host_info);
  for (auto& p : c->pool)
    for (auto e : p.ev) cudaEventDestroy(e);
  for (auto e : c->ag.ex)
    if (e) cudaGraphExecDestroy(e);
  if (c->cg.ex) cudaGraphExecDestroy(c->cg.ex);
  if (c->cyc) dfree(c, c->cyc);
  if (c->cyc_host) cudaFreeHost(c->cyc_host);
  if (c->comm && nccl().ok) {
    if (c->failed && nccl().CommAbort)
      nccl().CommAbort(c->comm);
    else
      nccl().CommDestroy(c->comm);
  }
  if (c->stream) cudaStreamSynchronize(c->stream);  // the stream-ordered frees have completed
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// (Re)load the point charges [nc][4] (host, validated): scaled SoA targets + records, raw copy,
// rank partition, exchange buffers, source/energy chunking, singular check (reading R11).
static bipb_status load_charges(bipb_ctx* c, int64_t nc, const std::vector<double>& Q) {
  double* olds[] = {c->qx, c->qy, c->qz, c->rec_ch, c->q4, c->phit, c->phi};
  for (double* p : olds)
    if (p) dfree(c, p);
  c->qx = c->qy = c->qz = c->rec_ch = c->q4 = c->phit = c->phi = nullptr;
  const int64_t ncm = std::max<int64_t>(nc, 1);
  std::vector<double> qxs(ncm, 0.0), qys(ncm, 0.0), qzs(ncm, 0.0), qrec(4 * ncm, 0.0), q4(4 * ncm, 0.0);
  for (int64_t k = 0; k < nc; ++k) {
    qxs[k] = Q[4 * k] * c->s; qys[k] = Q[4 * k + 1] * c->s; qzs[k] = Q[4 * k + 2] * c->s;
    qrec[4 * k] = qxs[k]; qrec[4 * k + 1] = qys[k]; qrec[4 * k + 2] = qzs[k]; qrec[4 * k + 3] = Q[4 * k + 3];
    for (int d = 0; d < 4; ++d) q4[4 * k + d] = Q[4 * k + d];
  }
  auto up = [&](double** d, const std::vector<double>& h) -> bipb_status {
    CK(dmalloc(c, d, h.size() * sizeof(double)));
    CK(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return BIPB_OK;
  };
  CKS(up(&c->qx, qxs)); CKS(up(&c->qy, qys)); CKS(up(&c->qz, qzs));
  CKS(up(&c->rec_ch, qrec)); CKS(up(&c->q4, q4));
  CK(dmalloc(c, &c->phit, ncm * sizeof(double)));
  CK(dmalloc(c, &c->phi, ncm * sizeof(double)));
  c->nc = nc;
  c->have_b = false;
  bipb_partition(nc, c->world, c->rank, &c->k0, &c->k1);
  c->kp = cdiv(ncm, c->world);
  if (c->sharded) {
    const int64_t st = std::max<int64_t>(2 * c->np, c->kp);
    if (st > c->stage_cap) {
      if (c->stage) dfree(c, c->stage);
      if (c->gather) dfree(c, c->gather);
      c->stage = c->gather = nullptr;
      CK(dmalloc(c, &c->stage, st * sizeof(double)));
      CK(dmalloc(c, &c->gather, (size_t)c->world * st * sizeof(double)));
      c->stage_cap = st;
    }
  }
  c->chunk_src = choose_chunk(c->n, ncm, SRC_TPB * SRC_T);
  c->nchunk_src = cdiv(ncm, c->chunk_src);
  c->chunk_en = choose_chunk_waves(ncm, c->n, EN_TPB * EN_T, c->en_resident);
  c->nchunk_en = cdiv(c->n, c->chunk_en);
  if (nc > 0) {  // a charge within 1e-6 A of a centroid (compared in scaled coordinates)
    CK(cudaMemsetAsync(c->dflag, 0, sizeof(int), c->stream));
    LAUNCH1D(min_dist_kernel, c->n, c->ex, c->ey, c->ez, c->n, c->rec_ch, nc, 1e-12 * c->s * c->s, c->dflag);
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, c->dflag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (flag) return fail(BIPB_ERR_SINGULAR, "a charge lies within 1e-6 A of an element centroid");
  }
  return BIPB_OK;
}

// Peer-store exchange (bipb_p2p.cuh): mailbox + flags in cudaMalloc memory (IPC-exportable),
// handles all-gathered once over the communicator, opened on every rank and SELF-TESTED before
// first use.  Devices are identified by UUID: ordinals are per process (under per-rank
// CUDA_VISIBLE_DEVICES every rank sees its own GPU as device 0).  Any failure on any rank -- a
// visible peer GPU without P2P access, an IPC handle that does not open, a probe word or flag that
// does not arrive -- is all-gathered, and then ALL ranks keep the NCCL collectives (auto) or setup
// fails (`require`: BIPB_DIST_P2P / BIPB_EXCHANGE=p2p).  BIPB_P2P_PROBE_FAIL=<rank> makes that
// rank report a failed probe (tests of the fallback).
static bipb_status p2p_setup(bipb_ctx* c, bool require) {
  if (c->world > P2P_MAX) {
    if (require) return fail(BIPB_ERR_ARG, "the peer-store exchange supports up to 16 ranks");
    return BIPB_OK;  // NCCL collectives
  }
  const int64_t m2 = 2 * c->n;
  c->p2p_stride = std::max<int64_t>((int64_t)c->world * 4 * m2, c->world);  // slots [world][R <= 4][2n]
  CK(cudaMalloc(&c->p2p_box, 2 * (size_t)c->p2p_stride * sizeof(double)));
  CK(cudaMalloc(&c->p2p_flags, (size_t)c->world * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(c->p2p_flags, 0, (size_t)c->world * sizeof(unsigned long long), c->stream));
  CK(cudaMemsetAsync(c->p2p_box, 0, (size_t)c->world * sizeof(unsigned long long), c->stream));
  if (!c->p2p_epoch) CK(dmalloc(c, &c->p2p_epoch, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(c->p2p_epoch, 0, sizeof(unsigned long long), c->stream));
  if (!c->p2p_err) {
    CK(cudaHostAlloc(&c->p2p_err, sizeof(unsigned int), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&c->p2p_err_dev, c->p2p_err, 0));
  }
  *c->p2p_err = 0u;
  c->boxes.p[c->rank] = c->p2p_box;
  c->flags.p[c->rank] = c->p2p_flags;
  if (c->world > 1) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    constexpr int W = 18;  // per rank: box handle (8 doubles), flags handle (8), device UUID (2)
    cudaIpcMemHandle_t hb, hf;
    CK(cudaIpcGetMemHandle(&hb, c->p2p_box));
    CK(cudaIpcGetMemHandle(&hf, c->p2p_flags));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, c->device));
    double mine[W];
    memcpy(mine, &hb, 64);
    memcpy(mine + 8, &hf, 64);
    memcpy(mine + 16, &prop.uuid, 16);
    double *dsend = nullptr, *drecv = nullptr;
    CK(dmalloc(c, &dsend, W * sizeof(double)));
    CK(dmalloc(c, &drecv, (size_t)c->world * W * sizeof(double)));
    std::vector<double> all((size_t)c->world * W);
    // all-gather of `cnt` doubles per rank; completes only once every rank reached it (a barrier)
    auto allgather = [&](const double* src, int cnt, double* dst) -> bipb_status {
      CK(cudaMemcpyAsync(dsend, src, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      CKS(nccl_check(c, nccl().AllGather(dsend, drecv, (size_t)cnt, ncclFloat64, c->comm, c->stream),
                     "ncclAllGather (p2p setup)"));
      CK(cudaMemcpyAsync(dst, drecv, (size_t)c->world * cnt * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CKS(ctx_sync(c));
      return BIPB_OK;
    };
    auto agree = [&](bool mine_ok, bool* all_ok) -> bipb_status {
      const double v = mine_ok ? 1.0 : 0.0;
      std::vector<double> oks((size_t)c->world);
      CKS(allgather(&v, 1, oks.data()));
      *all_ok = true;
      for (double o : oks) *all_ok = *all_ok && o != 0.0;
      return BIPB_OK;
    };
    CKS(allgather(mine, W, all.data()));
    // 1. reachability: peers on this GPU (same UUID) always; a peer GPU visible in this process
    // needs P2P access; a peer GPU not visible here is decided by the IPC open itself
    std::string why;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int q = 0; q < c->world && why.empty(); ++q) {
      if (q == c->rank || !memcmp(&all[(size_t)q * W + 16], mine + 16, 16)) continue;
      for (int d = 0; d < ndev; ++d) {
        cudaDeviceProp pd;
        if (cudaGetDeviceProperties(&pd, d) != cudaSuccess || memcmp(&pd.uuid, &all[(size_t)q * W + 16], 16)) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, c->device, d) != cudaSuccess || !can)
          why = "no P2P access to rank " + std::to_string(q) + "'s GPU";
      }
    }
    cudaGetLastError();
    // 2. open every peer's mailbox and flags
    for (int q = 0; q < c->world && why.empty(); ++q) {
      if (q == c->rank) continue;
      memcpy(&hb, &all[(size_t)q * W], 64);
      memcpy(&hf, &all[(size_t)q * W + 8], 64);
      void *pb = nullptr, *pf = nullptr;
      cudaError_t e1 = cudaIpcOpenMemHandle(&pb, hb, cudaIpcMemLazyEnablePeerAccess);
      if (e1 == cudaSuccess) c->p2p_opened.push_back(pb);
      cudaError_t e2 = e1 == cudaSuccess ? cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess) : e1;
      if (e1 == cudaSuccess && e2 == cudaSuccess) c->p2p_opened.push_back(pf);
      if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaGetLastError();
        why = "cudaIpcOpenMemHandle of rank " + std::to_string(q) + ": " +
              cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
        break;
      }
      c->boxes.p[q] = static_cast<double*>(pb);
      c->flags.p[q] = static_cast<unsigned long long*>(pf);
    }
    bool all_ok = false;
    CKS(agree(why.empty(), &all_ok));
    // 3. probe: every rank stores a known word into every mailbox and a flag into every flag
    // array; after a barrier each rank checks what arrived in its own memory
    if (all_ok) {
      const unsigned long long magic = 0x5EED000000000000ull;
      p2p_probe_kernel<<<1, 32, 0, c->stream>>>(c->boxes, c->flags, c->world, c->rank, magic);
      CK(cudaGetLastError());
      double dummy = 0.0;
      std::vector<double> bar((size_t)c->world);
      CKS(allgather(&dummy, 1, bar.data()));
      std::vector<unsigned long long> words((size_t)c->world), fl((size_t)c->world);
      CK(cudaMemcpyAsync(words.data(), c->p2p_box, (size_t)c->world * 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(fl.data(), c->p2p_flags, (size_t)c->world * 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int q = 0; q < c->world && why.empty(); ++q)
        if (words[q] != p2p_probe_word(q, c->rank) || fl[q] != magic + (unsigned long long)q)
          why = "probe from rank " + std::to_string(q) + " did not arrive";
      if (const char* pf = getenv("BIPB_P2P_PROBE_FAIL"))
        if (atoi(pf) == c->rank && why.empty()) why = "probe failure forced (BIPB_P2P_PROBE_FAIL)";
      CKS(agree(why.empty(), &all_ok));
    }
    if (!all_ok) {
      dfree(c, dsend);
      dfree(c, drecv);
      p2p_teardown(c);
      if (require)
        return fail(BIPB_ERR_NCCL, "BIPB_DIST_P2P: peer-store exchange unavailable" +
                                       (why.empty() ? std::string(" on another rank") : ": " + why));
      return BIPB_OK;  // NCCL collectives (c->p2p stays false)
    }
    // clean slate (probe words and flags) before a final barrier: no rank signals before every
    // rank has cleared its flags
    CK(cudaMemsetAsync(c->p2p_flags, 0, (size_t)c->world * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->p2p_box, 0, (size_t)c->world * sizeof(unsigned long long), c->stream));
    double dummy = 0.0;
    std::vector<double> bar((size_t)c->world);
    CKS(allgather(&dummy, 1, bar.data()));
    dfree(c, dsend);
    dfree(c, drecv);
  }
  CK(cudaStreamSynchronize(c->stream));
  c->p2p = true;
  return BIPB_OK;
}

static bipb_status setup_impl(bipb_ctx* c, int64_t n, const double* centroids, const double* normals,
                              const double* areas, int64_t nc, const double* charges, double eps1, double eps2,
                              double kappa, const bipb_dist* dist, void* cuda_stream) {
  Trace tr;
  // ---- host-side validation (bipb.h; SURVEY.md §8(b) "Errors")
  std::vector<double> C(3 * n), Nn(3 * n), W(n), Q(4 * std::max<int64_t>(nc, 0));
  auto fetch = [&](const double* src, double* dst, size_t cnt) -> bipb_status {
    if (cnt == 0) return BIPB_OK;
    if (is_device_ptr(src)) {
      CK(cudaMemcpy(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
      memcpy(dst, src, cnt * sizeof(double));
    }
    return BIPB_OK;
  };
  if (dist) {
    if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world) return fail(BIPB_ERR_ARG, "bad rank/world");
    if (dist->device >= 0) CK(cudaSetDevice(dist->device));
  }
  CK(cudaGetDevice(&c->device));
  pool_init_once(c->device);
  CKS(fetch(centroids, C.data(), 3 * n));
  CKS(fetch(normals, Nn.data(), 3 * n));
  CKS(fetch(areas, W.data(), n));
  CKS(fetch(charges, Q.data(), 4 * nc));
  if (!(eps1 > 0) || !(eps2 > 0) || !(kappa >= 0) || !std::isfinite(eps1) || !std::isfinite(eps2) ||
      !std::isfinite(kappa))
    return fail(BIPB_ERR_INPUT, "eps1, eps2 must be > 0 and kappa >= 0, finite");
  for (int64_t i = 0; i < n; ++i) {
    const double* x = &C[3 * i];
    const double* v = &Nn[3 * i];
    if (!std::isfinite(x[0]) || !std::isfinite(x[1]) || !std::isfinite(x[2]) || !std::isfinite(W[i]) ||
        !(W[i] > 0))
      return fail(BIPB_ERR_INPUT, "element " + std::to_string(i) + ": non-finite centroid or area <= 0");
    const double nn = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (!(std::fabs(nn - 1.0) <= 1e-6))
      return fail(BIPB_ERR_INPUT, "element " + std::to_string(i) + ": normal is not unit length");
  }
  for (int64_t k = 0; k < nc; ++k)
    for (int d = 0; d < 4; ++d)
      if (!std::isfinite(Q[4 * k + d])) return fail(BIPB_ERR_INPUT, "charge " + std::to_string(k) + " not finite");

  {  // exp table T[j] = 2^(-j/2^B), correctly rounded on the host (long double)
    double tab[EXP_TAB];
    for (int j = 0; j < EXP_TAB; ++j) tab[j] = (double)exp2l(-(long double)j / EXP_TAB);
    CK(cudaMemcpyToSymbol(g_exp_tab, tab, sizeof(tab)));
  }
  tr.mark("fetch + validate");
  c->n = n; c->nc = nc; c->eps1 = eps1; c->eps2 = eps2; c->kappa = kappa;
  c->eps = eps2 / eps1;  // reading R1
  c->pinv1 = 1.0 / (0.5 * (1.0 + c->eps));  // opt-in right preconditioner M^-1 (bipb_set_precond)
  c->pinv2 = 1.0 / (0.5 * (1.0 + 1.0 / c->eps));
  if (const char* pe = getenv("BIPB_PRECOND")) c->precond = (!strcmp(pe, "jacobi") || !strcmp(pe, "1")) ? 1 : 0;
  if (const char* se = getenv("BIPB_SUM")) c->sum_mode = (!strcmp(se, "fixed") || !strcmp(se, "0")) ? 0 : 1;
  if (const char* xb = getenv("BIPB_EXACT_BIAS")) c->xbias = atoi(xb);
  if (const char* e = getenv("BIPB_P2P_TIMEOUT_S")) c->p2p_timeout_ns = (unsigned long long)(atof(e) * 1e9);
  if (const char* e = getenv("BIPB_COMM_TIMEOUT_S")) c->comm_timeout_ns = (unsigned long long)(atof(e) * 1e9);
  c->screened = kappa > 0.0;
  c->s = c->screened ? kappa : 1.0;
  {  // resident energy-kernel CTAs on this device (whole-wave chunk rule, choose_chunk_waves)
    const size_t en_smem = sizeof(double) * STAGES * TILE * 8 + 8 * STAGES;
    int occ = 0, sms = 0, dev = 0;
    cudaError_t oe = cudaGetDevice(&dev);
    if (oe == cudaSuccess) oe = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (oe == cudaSuccess)
      oe = c->screened
               ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_kernel<ENERGY, EN_TPB, EN_T, true, EN_MINB>,
                                                               EN_TPB, en_smem)
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_kernel<ENERGY, EN_TPB, EN_T, false, EN_MINB>,
                                                               EN_TPB, en_smem);
    if (oe != cudaSuccess) {
      cudaGetLastError();
      occ = 0;  // unknown: the plain chunk rule
    }
    c->en_resident = (int64_t)sms * occ;
  }
  c->rank = dist ? dist->rank : 0;
  c->world = dist ? dist->world : 1;
  c->sharded = dist != nullptr;
  c->no_comm = dist && (dist->flags & BIPB_DIST_NO_COMM);
  bipb_partition(n, c->world, c->rank, &c->r0, &c->r1);
  c->np = cdiv(n, c->world);

  if (cuda_stream) {
    c->stream = (cudaStream_t)cuda_stream;
  } else {
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }

  tr.mark("stream + exp table");
  // ---- device layout: SoA elements (scaled), records, charges
  std::vector<double> sx(n), sy(n), sz(n), nx(n), ny(n), nz(n), rec(8 * n);
  for (int64_t i = 0; i < n; ++i) {
    sx[i] = C[3 * i] * c->s; sy[i] = C[3 * i + 1] * c->s; sz[i] = C[3 * i + 2] * c->s;
    nx[i] = Nn[3 * i]; ny[i] = Nn[3 * i + 1]; nz[i] = Nn[3 * i + 2];
    rec[8 * i] = sx[i]; rec[8 * i + 1] = sy[i]; rec[8 * i + 2] = sz[i];
    for (int d = 3; d < 8; ++d) rec[8 * i + d] = 0.0;
  }
  auto up = [&](double** d, const std::vector<double>& h) -> bipb_status {
    CK(dmalloc(c, d, h.size() * sizeof(double)));
    CK(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return BIPB_OK;
  };
  CKS(up(&c->ex, sx)); CKS(up(&c->ey, sy)); CKS(up(&c->ez, sz));
  CKS(up(&c->enx, nx)); CKS(up(&c->eny, ny)); CKS(up(&c->enz, nz));
  CKS(up(&c->ew, W)); CKS(up(&c->rec_el, rec));
  const int64_t m2 = 2 * n;
  CK(dmalloc(c, &c->b, m2 * sizeof(double)));
  CK(dmalloc(c, &c->ubuf, m2 * sizeof(double)));
  CK(dmalloc(c, &c->ybuf, m2 * sizeof(double)));
  CK(dmalloc(c, &c->xbuf, m2 * sizeof(double)));
  CK(dmalloc(c, &c->bbuf, m2 * sizeof(double)));
  CK(dmalloc(c, &c->tbuf, m2 * sizeof(double)));
  CK(dmalloc(c, &c->scal, 16 * sizeof(double)));
  CK(dmalloc(c, &c->red_part, RED_BLOCKS * sizeof(double)));
  CK(dmalloc(c, &c->red_cnt, sizeof(unsigned)));
  CK(cudaMemsetAsync(c->red_cnt, 0, sizeof(unsigned), c->stream));
  CK(dmalloc(c, &c->dflag, sizeof(int)));
  CK(cudaMallocHost(&c->host_info, 8 * sizeof(double)));
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, c->host_info) == cudaSuccess && pa.devicePointer)
      c->host_info_dev = static_cast<double*>(pa.devicePointer);
    cudaGetLastError();
  }
  {  // fused Arnoldi tail when the Krylov vectors fit one cluster's registers (BIPB_ARNOLDI=launches: off)
    const char* ae = getenv("BIPB_ARNOLDI");
    const bool force_off = ae && !strcmp(ae, "launches");
    c->arn_E = 0;
    if (!force_off)
      for (int E : {1, 2, 4, 8})
        if ((int64_t)ARN_CLUSTER * ARN_THREADS * E >= m2) {
          c->arn_E = E;
          break;
        }
  }

  tr.mark("upload + buffers");
  // ---- launch geometry (global sizes only => P-invariant sums)
  c->chunk_mv = choose_chunk(n, n, MV_TPB * MV_T);
  c->nchunk_mv = cdiv(n, c->chunk_mv);

  // ---- default matvec kernel: symmetric once there is >= 1 wave of (I, J) tiles, else the row
  // kernel (small problems); BIPB_MATVEC=row|sym overrides.  Symmetric buffers are allocated on
  // first use (sym_plan).
  {
    // r02 session 4: with the small block shape (B = 128) the symmetric kernel wins from C1 on
    // (C1 product 89 vs 107 us, C2 0.88 vs 1.36 ms); below SYM_MIN_TASKS small-shape tasks the row
    // kernel (profiles/r02/session4/small_sizes.jsonl)
    int64_t min_tasks = SYM_MIN_TASKS;
    if (const char* e = getenv("BIPB_SYM_MIN_TASKS")) min_tasks = atoll(e);  // tuning
    c->mv_kind = (sym_tasks(n, SymCfgSmall::TPB * SymCfgSmall::T) >= min_tasks) ? 1 : 0;
    const char* env = getenv("BIPB_MATVEC");
    if (env && (!strcmp(env, "row") || !strcmp(env, "0"))) c->mv_kind = 0;
    if (env && (!strcmp(env, "sym") || !strcmp(env, "1"))) c->mv_kind = 1;
    if (c->mv_kind == 1) {
      bipb_ctx::SymPlan* p;
      CKS(sym_plan<1>(c, &p));
    }
  }
  tr.mark("symmetric-kernel buffers");
  // ---- charges (layout, sharding, chunking, singular check)
  CKS(load_charges(c, nc, Q));
  tr.mark("singular check");
  // ---- NCCL communicator
  if (c->sharded && !c->no_comm) {
    NcclApi& api = nccl();
    if (!api.ok) return fail(BIPB_ERR_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    memcpy(&id, dist->nccl_uid, 128);
    CKS(nccl_check(c, api.CommInitRank(&c->comm, c->world, id, c->rank), "ncclCommInitRank"));
    // per-product exchange: peer stores (default when world > 1 and every rank can map every
    // peer) or NCCL collectives; flags BIPB_DIST_P2P / BIPB_DIST_NCCL and BIPB_EXCHANGE=p2p|nccl
    // force one
    int mode = (dist->flags & BIPB_DIST_P2P) ? 1 : ((dist->flags & BIPB_DIST_NCCL) ? 0 : 2);  // 2 = auto
    if (const char* e = getenv("BIPB_EXCHANGE")) {
      if (!strcmp(e, "p2p")) mode = 1;
      if (!strcmp(e, "nccl")) mode = 0;
    }
    if (mode == 1 || (mode == 2 && c->world > 1)) CKS(p2p_setup(c, mode == 1));
  }
  CK(cudaStreamSynchronize(c->stream));
  tr.mark("nccl + sync");
  return BIPB_OK;
}

bipb_status bipb_setup(bipb_ctx** out, int64_t n, const double* centroids, const double* normals,
                       const double* areas, int64_t nc, const double* charges, double eps1, double eps2,
                       double kappa, const bipb_dist* dist, void* cuda_stream) {
  g_err.clear();
  NvtxRange nvtx_("bipb_setup");
  if (!out) return fail(BIPB_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1) return fail(BIPB_ERR_ARG, "n must be >= 1");
  if (nc < 0) return fail(BIPB_ERR_ARG, "nc must be >= 0");
  if (!centroids || !normals || !areas || (nc > 0 && !charges)) return fail(BIPB_ERR_ARG, "NULL input array");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(BIPB_ERR_CUDA, "no CUDA device");
  }
  bipb_ctx* c = new bipb_ctx();
  bipb_status st = setup_impl(c, n, centroids, normals, areas, nc, charges, eps1, eps2, kappa, dist, cuda_stream);
  if (st != BIPB_OK) {
    std::string keep = g_err;
    bipb_destroy(c);
    g_err = keep;
    return st;
  }
  *out = c;
  return BIPB_OK;
}

bipb_status bipb_source(bipb_ctx* c, double* b) {
  NvtxRange nvtx_("bipb_source");
  if (!c) return fail(BIPB_ERR_ARG, "ctx is NULL");
  CKS(check_alive(c));
  const int64_t n = c->n;
  if (c->nc == 0) {
    CK(cudaMemsetAsync(c->b, 0, 2 * n * sizeof(double), c->stream));
  } else {
    const int64_t nloc = c->r1 - c->r0;
    PairArgs a{};
    a.tx = c->ex + c->r0; a.ty = c->ey + c->r0; a.tz = c->ez + c->r0;
    a.tnx = c->enx + c->r0; a.tny = c->eny + c->r0; a.tnz = c->enz + c->r0;
    a.tgt_begin = c->r0; a.ntgt = nloc;
    a.src = c->rec_ch; a.nsrc = c->nc; a.chunk = c->chunk_src;
    a.eps = c->eps; a.inveps = 1.0 / c->eps;
    a.sc1 = c->s; a.sc2 = c->s * c->s; a.sc3 = a.sc2 * c->s;
    CKS(ensure_part(c, (size_t)(2 * c->nchunk_src * std::max<int64_t>(nloc, 1))));
    a.part = c->part;
    CKS((launch_pair<SOURCE, SRC_TPB, SRC_T, SRC_MINB>(c, a, c->nchunk_src, 1)));
    const double scale = 1.0 / (FOUR_PI * c->eps1);
    if (!c->sharded) {
      LAUNCH1D(reduce_source_kernel, nloc, c->part, c->nchunk_src, nloc, scale, c->b, c->b + n);
    } else if (c->p2p) {
      LAUNCH1D(reduce_source_p2p_kernel, std::max<int64_t>(nloc, 1), c->part, c->nchunk_src, nloc, scale, c->r0, n,
               c->boxes, c->world, c->p2p_stride, c->p2p_epoch);
      CKS(p2p_publish_and_wait(c));
      LAUNCH1D(p2p_take_kernel, 2 * n, c->p2p_box, c->p2p_stride, c->p2p_epoch, 2 * n, c->b);
    } else {
      LAUNCH1D(reduce_source_kernel, nloc, c->part, c->nchunk_src, nloc, scale, c->stage, c->stage + c->np);
      CKS(allgather_rows(c, c->b));
    }
  }
  c->have_b = true;
  if (b) {
    CK(cudaMemcpyAsync(b, c->b, 2 * n * sizeof(double), cudaMemcpyDefault, c->stream));
  }
  CKS(ctx_sync(c));
  return BIPB_OK;
}

bipb_status bipb_matvec(bipb_ctx* c, const double* u, double* y) {
  NvtxRange nvtx_("bipb_matvec");
  if (!c || !u || !y) return fail(BIPB_ERR_ARG, "NULL argument");
  CKS(check_alive(c));
  if (u == y) return fail(BIPB_ERR_ARG, "u and y must not alias");
  const int64_t m2 = 2 * c->n;
  const double* ud;
  CKS(in_vec(c, u, m2, c->ubuf, &ud));
  bool ydev;
  CKS(vec_where(c, y, &ydev));
  double* yd = ydev ? y : c->ybuf;
  if (ydev && yd == ud) return fail(BIPB_ERR_ARG, "u and y must not alias");
  const bool exact = exact_active(c);
  CKS(matvec_dev(c, ud, yd));
  bool ovf = false;
  if (exact) CKS(exact_overflowed(c, &ovf));
  if (ovf) CKS(matvec_dev(c, ud, yd));  // out-of-range partial: the fixed-order double partials
  if (!ydev) CK(cudaMemcpyAsync(y, yd, m2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CKS(ctx_sync(c));
  return BIPB_OK;
}

// Y = A U for nrhs operands (device, [nrhs][2n]); symmetric kernel in passes of 4, 2, 1 operands,
// row kernel one by one.
static bipb_status matvec_batch_dev(bipb_ctx* c, int nrhs, const double* U, double* Y) {
  const int64_t m2 = 2 * c->n;
  int done = 0;
  while (done < nrhs) {
    const int left = nrhs - done;
    const double* u = U + (int64_t)done * m2;
    double* y = Y + (int64_t)done * m2;
    if (c->mv_kind == 0) {
      CKS(matvec_dev(c, u, y));
      done += 1;
    } else if (left >= 4) {
      CKS(matvec_sym_R<4>(c, u, y));
      done += 4;
    } else if (left >= 2) {
      CKS(matvec_sym_R<2>(c, u, y));
      done += 2;
    } else {
      CKS(matvec_sym_R<1>(c, u, y));
      done += 1;
    }
  }
  return BIPB_OK;
}

static bipb_status ensure_krylov(bipb_ctx* c, int m) {
  if (m <= c->m_cap) return BIPB_OK;
  double* bufs[] = {c->V, c->H, c->cs, c->sn, c->g, c->yk};
  for (double* p : bufs)
    if (p) dfree(c, p);
  c->V = c->H = c->cs = c->sn = c->g = c->yk = nullptr;
  c->m_cap = 0;
  CK(dmalloc(c, &c->V, (size_t)(m + 1) * 2 * c->n * sizeof(double)));
  CK(dmalloc(c, &c->H, (size_t)(m + 1) * m * sizeof(double)));
  CK(dmalloc(c, &c->cs, (size_t)m * sizeof(double)));
  CK(dmalloc(c, &c->sn, (size_t)m * sizeof(double)));
  CK(dmalloc(c, &c->g, (size_t)(m + 1) * sizeof(double)));
  CK(dmalloc(c, &c->yk, (size_t)m * sizeof(double)));
  if (!c->zbuf) CK(dmalloc(c, &c->zbuf, (size_t)2 * c->n * sizeof(double)));
  c->m_cap = m;
  return BIPB_OK;
}


// One Arnoldi step k of GMRES(m) on the context's Krylov arrays: w = A v_k;
// modified Gram-Schmidt; Givens update; the 16-byte residual record copied to pinned host
// memory; w /= h_{k+1,k} (harmless garbage on a happy breakdown: V[k+1] is then unused).
// Enqueue only (no synchronisation) so it can be captured as a CUDA graph.
static bipb_status enqueue_arnoldi_step(bipb_ctx* c, int k, int m, bool cycle = false) {
  const int64_t m2 = 2 * c->n;
  double* S = c->scal;
  double* vk = c->V + (int64_t)k * m2;
  double* w = c->V + (int64_t)(k + 1) * m2;
  if (c->precond) {  // right preconditioning: w = A M^-1 v_k
    LAUNCH1D(jacobi_scale_kernel, m2, c->zbuf, vk, c->n, c->pinv1, c->pinv2);
    CKS(matvec_dev(c, c->zbuf, w));
  } else {
    CKS(matvec_dev(c, vk, w));
  }
  if (c->arn_E > 0) {  // MGS + Givens + normalisation in one cluster kernel (bipb_vec.cuh)
    switch (c->arn_E) {
      case 1: arnoldi_fused_kernel<1><<<ARN_CLUSTER, ARN_THREADS, 0, c->stream>>>(c->V, m2, k, m, c->H, c->cs, c->sn, c->g, S, c->host_info_dev); break;
      case 2: arnoldi_fused_kernel<2><<<ARN_CLUSTER, ARN_THREADS, 0, c->stream>>>(c->V, m2, k, m, c->H, c->cs, c->sn, c->g, S, c->host_info_dev); break;
      case 4: arnoldi_fused_kernel<4><<<ARN_CLUSTER, ARN_THREADS, 0, c->stream>>>(c->V, m2, k, m, c->H, c->cs, c->sn, c->g, S, c->host_info_dev); break;
      default: arnoldi_fused_kernel<8><<<ARN_CLUSTER, ARN_THREADS, 0, c->stream>>>(c->V, m2, k, m, c->H, c->cs, c->sn, c->g, S, c->host_info_dev); break;
    }
    c->launches_all++;
    CK(cudaGetLastError());
    if (!c->host_info_dev && !cycle)
      CK(cudaMemcpyAsync(c->host_info, S + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    return BIPB_OK;
  }
  axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(w, nullptr, nullptr, c->V, m2, c->red_part, c->red_cnt,
                                                              c->H + 0 * m + k);
  c->launches_all++;
  for (int i = 0; i <= k; ++i) {
    const double* zi = (i < k) ? c->V + (int64_t)(i + 1) * m2 : w;
    double* outp = (i < k) ? c->H + (int64_t)(i + 1) * m + k : S + 2;
    axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(w, c->V + (int64_t)i * m2, c->H + (int64_t)i * m + k,
                                                                zi, m2, c->red_part, c->red_cnt, outp);
    c->launches_all++;
  }
  CK(cudaGetLastError());
  givens_kernel<<<1, 1, 0, c->stream>>>(c->H, c->cs, c->sn, c->g, S + 2, S + 3, k, m, S + 0, S + 6);
  c->launches_all++;
  if (!cycle) CK(cudaMemcpyAsync(c->host_info, S + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  LAUNCH1D(scale_div_kernel, m2, w, w, S + 3, m2);
  return BIPB_OK;
}

// Run step k: replay its CUDA graph when possible (no timing instrumentation active, the
// product's buffers warm), else enqueue eagerly; then wait and return (rel, h_{k+1,k}).
static bipb_status run_arnoldi_step(bipb_ctx* c, int k, int m, double* h2) {
  NvtxRange nvtx_("arnoldi_step");
  // opt-in (BIPB_GRAPHS=1): replay pays off only from the second solve in a context (measured:
  // C1 3.25 -> 2.82 ms per solve, C2 -2.6%, C3/C4 within noise; the first solve pays the capture)
  static const bool graphs_on = getenv("BIPB_GRAPHS") && !strcmp(getenv("BIPB_GRAPHS"), "1");
  const bool use = graphs_on && !c->timing && c->warm_kind == warm_key(c);
  if (use) {
    const int exact = exact_active(c) ? 1 : 0;  // the captured product differs per sum mode
    if (c->ag.V != c->V || c->ag.m != m || c->ag.kind != c->mv_kind || c->ag.precond != c->precond ||
        c->ag.exact != exact) {
      for (auto e : c->ag.ex)
        if (e) cudaGraphExecDestroy(e);
      c->ag.ex.assign(m, nullptr);
      c->ag.V = c->V;
      c->ag.m = m;
      c->ag.kind = c->mv_kind;
      c->ag.precond = c->precond;
      c->ag.exact = exact;
    }
    if (!c->ag.ex[k]) {
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      bipb_status st = enqueue_arnoldi_step(c, k, m);
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
      if (st != BIPB_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      if (ce != cudaSuccess) return fail(BIPB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      cudaGraphExec_t ex = nullptr;
      ce = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (ce != cudaSuccess) return fail(BIPB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
      c->ag.ex[k] = ex;
    }
    CK(cudaGraphLaunch(c->ag.ex[k], c->stream));
  } else {
    CKS(enqueue_arnoldi_step(c, k, m));
  }
  CKS(ctx_sync(c));
  h2[0] = c->host_info[0];
  h2[1] = c->host_info[1];
  return BIPB_OK;
}

// ---- device-side Arnoldi cycle (BIPB_GRAPHS=2): the m steps of a GMRES(m) cycle as ONE graph
// launch. Step k sits in an IF node on a condition that cycle_check_kernel clears when the host
// loop would leave the cycle after that step (breakdown, convergence, iteration cap, NaN), so the
// later steps do not run; the host reads the per-step records once per cycle instead of once per
// step. Single-GPU contexts only (the multi-rank exchange's collectives stay out of conditional
// bodies), after an eager product has prepared the product's buffers (capture cannot allocate).
static bool cycle_usable(const bipb_ctx* c) {
  static const bool on = getenv("BIPB_GRAPHS") && !strcmp(getenv("BIPB_GRAPHS"), "2");
  return on && !c->cycle_off && c->world == 1 && !c->timing && c->warm_kind == warm_key(c);
}

// Sink nodes of a graph (no dependents): the dependencies of the node appended after them.
static cudaError_t graph_sinks(cudaGraph_t g, std::vector<cudaGraphNode_t>& out) {
  out.clear();
  size_t n = 0;
  cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
  if (e != cudaSuccess || n == 0) return e;
  std::vector<cudaGraphNode_t> nodes(n);
  e = cudaGraphGetNodes(g, nodes.data(), &n);
  for (size_t i = 0; i < n && e == cudaSuccess; ++i) {
    size_t d = 0;
    e = cudaGraphNodeGetDependentNodes(nodes[i], nullptr, &d);
    if (e == cudaSuccess && d == 0) out.push_back(nodes[i]);
  }
  return e;
}

// The cycle graph: IF(c_0){ step 0; check 0; IF(c_1){ step 1; check 1; IF(c_2){ ... } } } -- the
// IF nodes are nested because a conditional handle belongs to ONE node: c_0 (top level) defaults
// to 1 at every launch, c_{k+1} is created in step k's body and always written by check k (1 to
// go on, 0 to leave the cycle), so no value from an earlier launch is ever read.
static bipb_status build_cycle_graph(bipb_ctx* c, int m) {
  const int exact = exact_active(c) ? 1 : 0;
  if (c->cg.ex && c->cg.V == c->V && c->cg.m == m && c->cg.kind == c->mv_kind && c->cg.precond == c->precond &&
      c->cg.exact == exact)
    return BIPB_OK;
  if (c->cg.ex) cudaGraphExecDestroy(c->cg.ex);
  c->cg.ex = nullptr;
  c->cg.V = nullptr;
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  bipb_status st = BIPB_OK;
  std::string what = "conditional handle 0";
  cudaGraphConditionalHandle cond = 0;
  cudaError_t ce = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
  cudaGraph_t parent = g;
  std::vector<cudaGraphNode_t> deps;
  for (int k = 0; k < m && ce == cudaSuccess && st == BIPB_OK; ++k) {
    what = "conditional node " + std::to_string(k);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node = nullptr;
    ce = cudaGraphAddNode(&node, parent, deps.empty() ? nullptr : deps.data(), deps.size(), &np);
    if (ce != cudaSuccess) break;
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaGraphConditionalHandle next = 0;
    if (k + 1 < m) {
      what = "conditional handle " + std::to_string(k + 1);
      ce = cudaGraphConditionalHandleCreate(&next, body, 0, 0);
      if (ce != cudaSuccess) break;
    }
    what = "begin capture " + std::to_string(k);
    ce = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) break;
    st = enqueue_arnoldi_step(c, k, m, true);
    if (st == BIPB_OK) {
      cycle_check_kernel<<<1, 1, 0, c->stream>>>(c->scal, c->cyc, k, next, k + 1 < m ? 1 : 0);
      ce = cudaGetLastError();
    }
    if (ce != cudaSuccess) what = "step capture " + std::to_string(k);
    cudaGraph_t captured = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(c->stream, &captured);
    if (ce == cudaSuccess && ee != cudaSuccess) {
      ce = ee;
      what = "end capture " + std::to_string(k);
    }
    if (ce == cudaSuccess) {
      what = "sinks " + std::to_string(k);
      ce = graph_sinks(body, deps);
    }
    parent = body;
    cond = next;
  }
  cudaGraphExec_t ex = nullptr;
  if (ce == cudaSuccess && st == BIPB_OK) {
    what = "instantiate";
    ce = cudaGraphInstantiate(&ex, g, 0);
  }
  cudaGraphDestroy(g);
  if (st != BIPB_OK) return st;
  if (ce != cudaSuccess) {
    cudaGetLastError();
    return fail(BIPB_ERR_CUDA, "cycle graph (" + what + "): " + cudaGetErrorString(ce));
  }
  c->cg.ex = ex;
  c->cg.V = c->V;
  c->cg.m = m;
  c->cg.kind = c->mv_kind;
  c->cg.precond = c->precond;
  c->cg.exact = exact;
  return BIPB_OK;
}

// One cycle on the device: parameters in, the graph, the per-step records (rel, h_{k+1,k}) out
// into c->cyc_host[8 ..]; the caller replays the host loop's bookkeeping on them.
static bipb_status run_cycle(bipb_ctx* c, int m, double beta_b, double tol, int64_t its, int max_iters, bool exact,
                             bool* ran) {
  NvtxRange nvtx_("arnoldi_cycle");
  *ran = false;
  if (c->cyc_cap < m) {
    if (c->cyc) dfree(c, c->cyc);
    if (c->cyc_host) cudaFreeHost(c->cyc_host);
    c->cyc = nullptr;
    c->cyc_host = nullptr;
    c->cyc_cap = 0;
    CK(dmalloc(c, &c->cyc, (size_t)(8 + 2 * m) * sizeof(double)));
    CK(cudaMallocHost(&c->cyc_host, (size_t)(8 + 2 * m) * sizeof(double)));
    c->cyc_cap = m;
    if (c->cg.ex) cudaGraphExecDestroy(c->cg.ex);  // it holds the old c->cyc
    c->cg.ex = nullptr;
  }
  if (build_cycle_graph(c, m) != BIPB_OK) {  // e.g. a node type the driver rejects in a conditional body
    c->cycle_off = true;
    c->cycle_err = g_err;
    if (getenv("BIPB_CYCLE_VERBOSE")) fprintf(stderr, "[bipb] cycle graphs off: %s\n", g_err.c_str());
    return BIPB_OK;  // the caller runs this cycle eagerly
  }
  double* h = c->cyc_host;
  h[0] = beta_b;
  h[1] = tol;
  h[2] = (double)its;
  h[3] = (double)max_iters;
  h[4] = exact ? 1.0 : 0.0;
  CK(cudaMemcpyAsync(c->cyc, h, 8 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaGraphLaunch(c->cg.ex, c->stream));
  CK(cudaMemcpyAsync(h + 8, c->cyc + 8, 2 * m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CKS(ctx_sync(c));
  *ran = true;
  c->graph_cycles++;
  return BIPB_OK;
}

// ---- multi-RHS GMRES: nrhs independent GMRES(m) runs in lockstep,
// each exactly the algorithm of bipb_gmres_solve; every Arnoldi step applies A to all systems
// still iterating through one batched (shared-pair) product.
struct GmresSys {
  double *V = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr, *yk = nullptr, *S = nullptr;
  const double* b = nullptr;
  double* x = nullptr;
  double beta_b = 0.0, rel = 1.0;
  int64_t its = 0, restarts = 0, matvecs = 0, hl = 0;
  int kdone = 0;
  bool converged = false, finished = false, in_cycle = false, first = true;
  bipb_report* rep = nullptr;
};

static bipb_status gmres_batch_impl(bipb_ctx* c, int R, const double* const* bd, double* const* xd, int m, double tol,
                                    int max_iters, int check_true, bipb_report* reps, int* n_not_conv) {
  const int64_t m2 = 2 * c->n;
  std::vector<GmresSys> sy(R);
  std::vector<double*> owned;
  auto alloc = [&](double** p, size_t cnt) -> bipb_status {
    CK(dmalloc(c, p, cnt * sizeof(double)));
    owned.push_back(*p);
    return BIPB_OK;
  };
  struct Guard {
    bipb_ctx* c;
    std::vector<double*>* v;
    ~Guard() {
      for (double* p : *v) dfree(c, p);
    }
  } guard{c, &owned};
  double *U = nullptr, *Y = nullptr;
  CKS(alloc(&U, (size_t)R * m2));
  CKS(alloc(&Y, (size_t)R * m2));
  for (int r = 0; r < R; ++r) {
    GmresSys& q = sy[r];
    q.b = bd[r];
    q.x = xd[r];
    q.rep = reps ? reps + r : nullptr;
    CKS(alloc(&q.V, (size_t)(m + 1) * m2));
    CKS(alloc(&q.H, (size_t)(m + 1) * m));
    CKS(alloc(&q.cs, (size_t)m));
    CKS(alloc(&q.sn, (size_t)m));
    CKS(alloc(&q.g, (size_t)(m + 1)));
    CKS(alloc(&q.yk, (size_t)m));
    CKS(alloc(&q.S, 16));
    CKS(dot_dev(c, q.b, q.b, m2, 1.0, q.S + 0));
    LAUNCH1D(sqrt_kernel, 1, q.S + 0, q.S + 0);
  }
  double h2[2];
  for (int r = 0; r < R; ++r) {
    CKS(read_scalars(c, sy[r].S, 1, h2));
    sy[r].beta_b = h2[0];
    if (h2[0] == 0.0) {
      CK(cudaMemsetAsync(sy[r].x, 0, m2 * sizeof(double), c->stream));
      sy[r].converged = sy[r].finished = true;
      sy[r].rel = 0.0;
    }
  }
  // batched A applied to the listed systems' vectors src(q) -> dst(q)
  auto apply = [&](std::vector<int>& list, auto src, auto dst, bool arnoldi = false) -> bipb_status {
    const int k = (int)list.size();
    if (k == 0) return BIPB_OK;
    for (int t = 0; t < k; ++t) {
      if (arnoldi && c->precond) {  // right preconditioning: the operand is M^-1 v_k
        LAUNCH1D(jacobi_scale_kernel, m2, U + t * m2, src(sy[list[t]]), c->n, c->pinv1, c->pinv2);
      } else {
        CK(cudaMemcpyAsync(U + t * m2, src(sy[list[t]]), m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    CKS(matvec_batch_dev(c, k, U, Y));
    for (int t = 0; t < k; ++t) {
      CK(cudaMemcpyAsync(dst(sy[list[t]]), Y + t * m2, m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      sy[list[t]].matvecs++;
    }
    return BIPB_OK;
  };
  for (;;) {
    // ---- cycle start: r = b - A x for every unfinished system (x = 0: r = b, no product)
    std::vector<int> need, act;
    for (int r = 0; r < R; ++r) {
      GmresSys& q = sy[r];
      if (q.finished) continue;
      CKS(dot_dev(c, q.x, q.x, m2, 1.0, q.S + 4));
      CKS(read_scalars(c, q.S + 4, 1, h2));
      if (h2[0] == 0.0) {
        CK(cudaMemcpyAsync(q.V, q.b, m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      } else {
        need.push_back(r);
      }
      act.push_back(r);
    }
    if (act.empty()) break;
    CKS(apply(need, [](GmresSys& q) { return (const double*)q.x; }, [](GmresSys& q) { return q.V; }));
    for (int r : need) LAUNCH1D(residual_kernel, m2, sy[r].V, sy[r].b, sy[r].V, m2);
    std::vector<int> iter;
    for (int r : act) {
      GmresSys& q = sy[r];
      if (!q.first) ++q.restarts;
      q.first = false;
      CKS(dot_dev(c, q.V, q.V, m2, 1.0, q.S + 1));
      LAUNCH1D(sqrt_kernel, 1, q.S + 1, q.S + 1);
      CKS(read_scalars(c, q.S + 1, 1, h2));
      q.rel = h2[0] / q.beta_b;
      if (q.rel <= tol) { q.converged = q.finished = true; continue; }
      if (q.its >= max_iters) { q.finished = true; continue; }
      LAUNCH1D(scale_div_kernel, m2, q.V, q.V, q.S + 1, m2);
      init_g_kernel<<<1, 32, 0, c->stream>>>(q.g, q.S + 1, m);
      c->launches_all++;
      q.kdone = 0;
      q.in_cycle = true;
      iter.push_back(r);
    }
    // ---- Arnoldi steps in lockstep
    for (int k = 0; k < m && !iter.empty(); ++k) {
      CKS(apply(iter, [k, m2](GmresSys& q) { return (const double*)(q.V + (int64_t)k * m2); },
                [k, m2](GmresSys& q) { return q.V + (int64_t)(k + 1) * m2; }, true));
      std::vector<int> next;
      for (int r : iter) {
        GmresSys& q = sy[r];
        q.its++;
        double* w = q.V + (int64_t)(k + 1) * m2;
        axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(w, nullptr, nullptr, q.V, m2, c->red_part,
                                                                    c->red_cnt, q.H + k);
        c->launches_all++;
        for (int i = 0; i <= k; ++i) {
          const double* zi = (i < k) ? q.V + (int64_t)(i + 1) * m2 : w;
          double* outp = (i < k) ? q.H + (int64_t)(i + 1) * m + k : q.S + 2;
          axpy_dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(w, q.V + (int64_t)i * m2, q.H + (int64_t)i * m + k,
                                                                      zi, m2, c->red_part, c->red_cnt, outp);
          c->launches_all++;
        }
        givens_kernel<<<1, 1, 0, c->stream>>>(q.H, q.cs, q.sn, q.g, q.S + 2, q.S + 3, k, m, q.S + 0, q.S + 6);
        c->launches_all++;
        CK(cudaGetLastError());
        CKS(read_scalars(c, q.S + 6, 2, h2));
        q.rel = h2[0];
        if (q.rep && q.rep->history && q.hl < q.rep->history_cap) q.rep->history[q.hl] = q.rel;
        ++q.hl;
        q.kdone = k + 1;
        if (h2[1] <= 1e-14 * q.beta_b) continue;  // happy breakdown: leaves the cycle
        LAUNCH1D(scale_div_kernel, m2, w, w, q.S + 3, m2);
        if (q.rel <= tol || q.its >= max_iters) continue;
        next.push_back(r);
      }
      iter.swap(next);
    }
    // ---- end of cycle: x += V y for the systems that iterated
    for (int r = 0; r < R; ++r) {
      GmresSys& q = sy[r];
      if (!q.in_cycle) continue;
      q.in_cycle = false;
      backsolve_kernel<<<1, 1, 0, c->stream>>>(q.H, q.g, q.yk, q.kdone, m);
      c->launches_all++;
      if (c->precond)
        LAUNCH1D(update_x_prec_kernel, m2, q.x, q.V, q.yk, q.kdone, c->n, c->pinv1, c->pinv2);
      else
        LAUNCH1D(update_x_kernel, m2, q.x, q.V, q.yk, q.kdone, m2);
      if (q.rel <= tol) q.converged = q.finished = true;
      else if (q.its >= max_iters) q.finished = true;
    }
  }
  if (check_true) {
    std::vector<int> all;
    for (int r = 0; r < R; ++r)
      if (sy[r].beta_b != 0.0) all.push_back(r);
    CKS(apply(all, [](GmresSys& q) { return (const double*)q.x; }, [](GmresSys& q) { return q.V; }));
    for (int r : all) {
      GmresSys& q = sy[r];
      LAUNCH1D(residual_kernel, m2, q.V, q.b, q.V, m2);
      CKS(dot_dev(c, q.V, q.V, m2, 1.0, q.S + 4));
      LAUNCH1D(sqrt_kernel, 1, q.S + 4, q.S + 4);
      CKS(read_scalars(c, q.S + 4, 1, h2));
      if (q.rep) q.rep->rel_res_true = h2[0] / q.beta_b;
    }
  }
  CKS(ctx_sync(c));
  *n_not_conv = 0;
  for (int r = 0; r < R; ++r) {
    GmresSys& q = sy[r];
    if (!q.converged) ++*n_not_conv;
    if (q.rep) {
      q.rep->iterations = q.its;
      q.rep->restarts = q.restarts;
      q.rep->matvecs = q.matvecs;
      q.rep->converged = q.converged ? 1 : 0;
      q.rep->rel_res_est = q.rel;
      q.rep->history_len = q.hl;
      if (!check_true) q.rep->rel_res_true = (q.beta_b == 0.0) ? 0.0 : -1.0;
    }
  }
  return BIPB_OK;
}

bipb_status bipb_gmres_solve(bipb_ctx* c, const double* b, double* x, int32_t restart_m, double tol,
                             int32_t max_iters, int32_t check_true, bipb_report* rep) {
  NvtxRange nvtx_("bipb_gmres_solve");
  if (!c || !x) return fail(BIPB_ERR_ARG, "NULL argument");
  if (restart_m < 1 || max_iters < 1 || !(tol > 0)) return fail(BIPB_ERR_ARG, "restart_m, max_iters >= 1, tol > 0");
  CKS(check_alive(c));
  if (!b && !c->have_b) return fail(BIPB_ERR_ARG, "b is NULL and bipb_source has not been called");
  const int64_t m2 = 2 * c->n;
  const int m = restart_m;
  CKS(ensure_krylov(c, m));
  const double* bd = c->b;
  if (b) CKS(in_vec(c, b, m2, c->bbuf, &bd));
  bool xdev;
  CKS(vec_where(c, x, &xdev));
  double* xd = xdev ? x : c->xbuf;
  if (!xdev) CK(cudaMemcpyAsync(xd, x, m2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  double* S = c->scal;  // [0] ||b||, [1] beta, [2] hk1sq, [3] hk1, [4] ||x||^2
  int64_t its = 0, restarts = 0, matvecs = 0, hl = 0;
  bool converged = false;
  double rel = 1.0, h2[2];
  if (rep) rep->rel_res_true = -1.0;
  // exact sums: an out-of-range partial (NaN product, bipb_exact.cuh) restarts the solve from x0
  // with the fixed-order double partials
  const bool exact = exact_active(c);
  if (exact) {
    if (!c->x0save) CK(dmalloc(c, &c->x0save, m2 * sizeof(double)));
    CK(cudaMemcpyAsync(c->x0save, xd, m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
rerun:
  its = restarts = matvecs = hl = 0;
  converged = false;
  rel = 1.0;

  CKS(dot_dev(c, bd, bd, m2, 1.0, S + 0));
  LAUNCH1D(sqrt_kernel, 1, S + 0, S + 0);
  CKS(read_scalars(c, S, 1, h2));
  const double beta_b = h2[0];
  if (beta_b == 0.0) {
    CK(cudaMemsetAsync(xd, 0, m2 * sizeof(double), c->stream));
    converged = true;
    rel = 0.0;
    if (rep) rep->rel_res_true = 0.0;
  } else {
    bool first = true;
    for (;;) {
      // r = b - A x  (x = 0 => r = b without a product), into V[0]
      CKS(dot_dev(c, xd, xd, m2, 1.0, S + 4));
      CKS(read_scalars(c, S + 4, 1, h2));
      if (h2[0] == 0.0) {
        CK(cudaMemcpyAsync(c->V, bd, m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      } else {
        CKS(matvec_dev(c, xd, c->tbuf));
        ++matvecs;
        LAUNCH1D(residual_kernel, m2, c->V, bd, c->tbuf, m2);
      }
      if (!first) ++restarts;
      first = false;
      CKS(dot_dev(c, c->V, c->V, m2, 1.0, S + 1));
      LAUNCH1D(sqrt_kernel, 1, S + 1, S + 1);
      CKS(read_scalars(c, S + 1, 1, h2));
      rel = h2[0] / beta_b;
      if (rel <= tol) { converged = true; break; }
      if (its >= max_iters) break;
      LAUNCH1D(scale_div_kernel, m2, c->V, c->V, S + 1, m2);
      init_g_kernel<<<1, 32, 0, c->stream>>>(c->g, S + 1, m);
      c->launches_all++;
      int kdone = 0;
      bool cycle = false;
      if (cycle_usable(c)) CKS(run_cycle(c, m, beta_b, tol, its, max_iters, exact, &cycle));
      for (int k = 0; k < m; ++k) {
        if (cycle) {
          h2[0] = c->cyc_host[8 + 2 * k];
          h2[1] = c->cyc_host[9 + 2 * k];
        } else {
          CKS(run_arnoldi_step(c, k, m, h2));
        }
        ++matvecs;
        ++its;
        rel = h2[0];
        const double hk1 = h2[1];
        if (rep && rep->history && hl < rep->history_cap) rep->history[hl] = rel;
        ++hl;
        kdone = k + 1;
        if (hk1 <= 1e-14 * beta_b) break;  // happy breakdown
        if (rel <= tol || its >= max_iters) break;
        if (exact && !(rel == rel)) break;
      }
      backsolve_kernel<<<1, 1, 0, c->stream>>>(c->H, c->g, c->yk, kdone, m);
      c->launches_all++;
      if (c->precond)
        LAUNCH1D(update_x_prec_kernel, m2, xd, c->V, c->yk, kdone, c->n, c->pinv1, c->pinv2);
      else
        LAUNCH1D(update_x_kernel, m2, xd, c->V, c->yk, kdone, m2);
      if (rel <= tol) { converged = true; break; }
      if (its >= max_iters) break;
      if (exact && !(rel == rel)) break;
    }
    if (check_true) {
      CKS(matvec_dev(c, xd, c->tbuf));
      ++matvecs;
      LAUNCH1D(residual_kernel, m2, c->tbuf, bd, c->tbuf, m2);
      CKS(dot_dev(c, c->tbuf, c->tbuf, m2, 1.0, S + 4));
      LAUNCH1D(sqrt_kernel, 1, S + 4, S + 4);
      CKS(read_scalars(c, S + 4, 1, h2));
      if (rep) rep->rel_res_true = h2[0] / beta_b;
    }
  }
  if (exact && c->sum_mode == 1 && !c->exact_off) {
    bool ovf = false;
    CKS(exact_overflowed(c, &ovf));
    if (ovf) {
      CK(cudaMemcpyAsync(xd, c->x0save, m2 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      goto rerun;
    }
  }
  if (!xdev) CK(cudaMemcpyAsync(x, xd, m2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CKS(ctx_sync(c));
  if (rep) {
    rep->iterations = its;
    rep->restarts = restarts;
    rep->matvecs = matvecs;
    rep->converged = converged ? 1 : 0;
    rep->rel_res_est = rel;
    rep->history_len = hl;
  }
  if (!converged) return fail(BIPB_NOT_CONVERGED, "GMRES reached max_iters");
  return BIPB_OK;
}


bipb_status bipb_gmres_solve_batch(bipb_ctx* c, int32_t nrhs, const double* B, double* X, int32_t restart_m,
                                   double tol, int32_t max_iters, int32_t check_true, bipb_report* reps) {
  NvtxRange nvtx_("bipb_gmres_solve_batch");
  if (!c || !B || !X || nrhs < 1) return fail(BIPB_ERR_ARG, "NULL argument or nrhs < 1");
  CKS(check_alive(c));
  if (restart_m < 1 || max_iters < 1 || !(tol > 0)) return fail(BIPB_ERR_ARG, "restart_m, max_iters >= 1, tol > 0");
  const int64_t m2 = 2 * c->n;
  bool bdev, xdev;
  CKS(vec_where(c, B, &bdev));
  CKS(vec_where(c, X, &xdev));
  double *bst = nullptr, *xst = nullptr;
  if (!bdev) {
    CK(dmalloc(c, &bst, (size_t)nrhs * m2 * sizeof(double)));
    CK(cudaMemcpyAsync(bst, B, (size_t)nrhs * m2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  if (!xdev) {
    CK(dmalloc(c, &xst, (size_t)nrhs * m2 * sizeof(double)));
    CK(cudaMemcpyAsync(xst, X, (size_t)nrhs * m2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  std::vector<const double*> bp(nrhs);
  std::vector<double*> xp(nrhs);
  for (int r = 0; r < nrhs; ++r) {
    bp[r] = (bdev ? B : bst) + (int64_t)r * m2;
    xp[r] = (xdev ? X : xst) + (int64_t)r * m2;
  }
  int not_conv = 0;
  bipb_status st = gmres_batch_impl(c, nrhs, bp.data(), xp.data(), restart_m, tol, max_iters, check_true, reps,
                                    &not_conv);
  if (st == BIPB_OK && !xdev)
    CK(cudaMemcpyAsync(X, xst, (size_t)nrhs * m2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (st == BIPB_OK) st = ctx_sync(c);
  else cudaStreamSynchronize(c->stream);
  if (bst) dfree(c, bst);
  if (xst) dfree(c, xst);
  if (st != BIPB_OK) return st;
  if (not_conv) return fail(BIPB_NOT_CONVERGED, std::to_string(not_conv) + " system(s) reached max_iters");
  return BIPB_OK;
}

bipb_status bipb_energy(bipb_ctx* c, const double* x, double* e_sol, double* phi_reac) {
  NvtxRange nvtx_("bipb_energy");
  if (!c || !x || !e_sol) return fail(BIPB_ERR_ARG, "NULL argument");
  CKS(check_alive(c));
  const int64_t n = c->n, nc = c->nc, m2 = 2 * n;
  double e = 0.0;
  if (nc > 0) {
    const double* xd;
    CKS(in_vec(c, x, m2, c->ubuf, &xd));
    LAUNCH1D(prescale_kernel, n, xd, c->ew, c->enx, c->eny, c->enz, c->rec_el, n);
    const int64_t kloc = c->k1 - c->k0;
    PairArgs a{};
    a.tx = c->qx + c->k0; a.ty = c->qy + c->k0; a.tz = c->qz + c->k0;
    a.tgt_begin = c->k0; a.ntgt = kloc;
    a.src = c->rec_el; a.nsrc = n; a.chunk = c->chunk_en;
    a.eps = c->eps; a.inveps = 1.0 / c->eps;
    a.sc1 = c->s; a.sc2 = c->s * c->s; a.sc3 = a.sc2 * c->s;
    CKS(ensure_part(c, (size_t)(2 * c->nchunk_en * std::max<int64_t>(kloc, 1))));
    a.part = c->part;
    CKS((launch_pair<ENERGY, EN_TPB, EN_T, EN_MINB>(c, a, c->nchunk_en, 2)));
    if (!c->sharded) {
      LAUNCH1D(reduce_energy_kernel, kloc, c->part, c->nchunk_en, kloc, c->phit);
    } else if (c->p2p && nc <= c->p2p_stride) {
      LAUNCH1D(reduce_energy_p2p_kernel, std::max<int64_t>(kloc, 1), c->part, c->nchunk_en, kloc, c->k0, c->boxes,
               c->world, c->p2p_stride, c->p2p_epoch);
      CKS(p2p_publish_and_wait(c));
      LAUNCH1D(p2p_take_kernel, nc, c->p2p_box, c->p2p_stride, c->p2p_epoch, nc, c->phit);
    } else {
      LAUNCH1D(reduce_energy_kernel, kloc, c->part, c->nchunk_en, kloc, c->stage);
      if (c->no_comm) {
        CK(cudaMemsetAsync(c->gather, 0, (size_t)c->world * c->kp * sizeof(double), c->stream));
        CK(cudaMemcpyAsync(c->gather + (size_t)c->rank * c->kp, c->stage, kloc * sizeof(double),
                           cudaMemcpyDeviceToDevice, c->stream));
      } else {
        CKS(nccl_check(c, nccl().AllGather(c->stage, c->gather, (size_t)c->kp, ncclFloat64, c->comm, c->stream),
                       "ncclAllGather"));
      }
      LAUNCH1D(unpack1_kernel, c->world * c->kp, c->gather, nc, c->kp, c->world, c->phit);
    }
    energy_sum_kernel<<<RED_BLOCKS, RED_THREADS, 0, c->stream>>>(c->q4, c->phit, nc, c->red_part, c->red_cnt,
                                                                  c->scal + 5);
    c->launches_all++;
    CK(cudaGetLastError());
    double h[1];
    CKS(read_scalars(c, c->scal + 5, 1, h));
    e = h[0];
    if (phi_reac) {
      LAUNCH1D(phi_scale_kernel, nc, c->phit, c->phi, nc);
      CK(cudaMemcpyAsync(phi_reac, c->phi, nc * sizeof(double), cudaMemcpyDefault, c->stream));
    }
  }
  CK(cudaMemcpyAsync(e_sol, &e, sizeof(double), cudaMemcpyDefault, c->stream));
  CKS(ctx_sync(c));
  return BIPB_OK;
}

bipb_status bipb_matvec_batch(bipb_ctx* c, int32_t nrhs, const double* U, double* Y) {
  NvtxRange nvtx_("bipb_matvec_batch");
  if (!c || !U || !Y || nrhs < 1) return fail(BIPB_ERR_ARG, "bad argument");
  CKS(check_alive(c));
  const int64_t m2 = 2 * c->n;
  bool udev, ydev;
  CKS(vec_where(c, U, &udev));
  CKS(vec_where(c, Y, &ydev));
  // host operands are staged through device buffers in slices of up to 4 operands
  const int64_t slice = (udev && ydev) ? nrhs : 4;
  if (!(udev && ydev) && !c->bat_U) {
    CK(dmalloc(c, &c->bat_U, (size_t)4 * m2 * sizeof(double)));
    CK(dmalloc(c, &c->bat_Y, (size_t)4 * m2 * sizeof(double)));
  }
  for (int64_t r0 = 0; r0 < nrhs; r0 += slice) {
    const int k = (int)std::min<int64_t>(slice, nrhs - r0);
    const double* ud = U + r0 * m2;
    double* yd = Y + r0 * m2;
    if (!udev) {
      CK(cudaMemcpyAsync(c->bat_U, ud, (size_t)k * m2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      ud = c->bat_U;
    }
    double* yk = ydev ? yd : c->bat_Y;
    if (yk == ud) return fail(BIPB_ERR_ARG, "U and Y must not alias");
    CKS(matvec_batch_dev(c, k, ud, yk));
    if (!ydev) CK(cudaMemcpyAsync(yd, yk, (size_t)k * m2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  CKS(ctx_sync(c));
  return BIPB_OK;
}

bipb_status bipb_set_charges(bipb_ctx* c, int64_t nc, const double* charges) {
  if (!c || nc < 0 || (nc > 0 && !charges)) return fail(BIPB_ERR_ARG, "bad argument");
  CKS(check_alive(c));
  std::vector<double> Q(4 * std::max<int64_t>(nc, 0));
  if (nc > 0) {
    if (is_device_ptr(charges)) {
      CK(cudaMemcpy(Q.data(), charges, Q.size() * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
      memcpy(Q.data(), charges, Q.size() * sizeof(double));
    }
  }
  for (size_t k = 0; k < Q.size(); ++k)
    if (!std::isfinite(Q[k])) return fail(BIPB_ERR_INPUT, "charge " + std::to_string(k / 4) + " not finite");
  CKS(load_charges(c, nc, Q));
  CK(cudaStreamSynchronize(c->stream));
  return BIPB_OK;
}

bipb_status bipb_set_matvec_kernel(bipb_ctx* c, int32_t kind) {
  if (!c || (kind != 0 && kind != 1)) return fail(BIPB_ERR_ARG, "kind must be 0 (row) or 1 (symmetric)");
  c->mv_kind = kind;
  return BIPB_OK;
}

int32_t bipb_get_matvec_kernel(bipb_ctx* c) { return c ? c->mv_kind : -1; }

int32_t bipb_get_arnoldi(bipb_ctx* c) { return c ? c->arn_E : -1; }

int64_t bipb_get_graph_cycles(bipb_ctx* c) { return c ? c->graph_cycles : -1; }

bipb_status bipb_set_precond(bipb_ctx* c, int32_t kind) {
  if (!c) return fail(BIPB_ERR_ARG, "ctx is NULL");
  if (kind != 0 && kind != 1) return fail(BIPB_ERR_ARG, "precond kind must be 0 (none) or 1 (jump-term diagonal)");
  c->precond = kind;
  return BIPB_OK;
}
int32_t bipb_get_precond(bipb_ctx* c) { return c ? c->precond : -1; }

bipb_status bipb_set_sum_mode(bipb_ctx* c, int32_t mode) {
  if (!c) return fail(BIPB_ERR_ARG, "ctx is NULL");
  if (mode != 0 && mode != 1) return fail(BIPB_ERR_ARG, "sum mode must be 0 (fixed-order doubles) or 1 (exact)");
  c->sum_mode = mode;
  c->exact_off = false;
  return BIPB_OK;
}
int32_t bipb_get_sum_mode(bipb_ctx* c) {
  if (!c) return -1;
  return exact_active(c) ? 1 : 0;
}

int32_t bipb_get_exchange(bipb_ctx* c) {
  if (!c) return -1;
  if (!c->sharded || c->no_comm) return 0;
  return c->p2p ? 2 : 1;
}

bipb_status bipb_timing_enable(bipb_ctx* c, int32_t on) {
  if (!c) return fail(BIPB_ERR_ARG, "ctx is NULL");
  c->timing = on != 0;
  return BIPB_OK;
}

bipb_status bipb_timing_reset(bipb_ctx* c) {
  if (!c) return fail(BIPB_ERR_ARG, "ctx is NULL");
  CK(cudaStreamSynchronize(c->stream));
  for (auto& p : c->pool) {
    p.used = 0;
    p.launches = 0;
  }
  c->launches_all = 0;
  return BIPB_OK;
}

bipb_status bipb_timing_get(bipb_ctx* c, int32_t which, double* total_ms, int64_t* launches) {
  if (!c || which < 0 || which > 3) return fail(BIPB_ERR_ARG, "bad argument");
  CK(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  int64_t cnt = 0;
  if (which == 3) {
    cnt = c->launches_all;
  } else {
    EventPool& p = c->pool[which];
    for (size_t i = 0; i + 1 < p.used; i += 2) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, p.ev[i], p.ev[i + 1]));
      tot += ms;
    }
    cnt = p.launches;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = cnt;
  return BIPB_OK;
}

}  // extern "C"

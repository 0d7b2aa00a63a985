// csc_api.cu -- the C ABI (include/csc.h) over the sm_100a kernels.
//
// Iteration structure (Alg.1):
//   csc_code_step   [r cache invalid -> dense residual] -> [tau_z = 1/L_D] -> mask -> masked step
//   csc_filter_step dense residual r' -> Z^T r' -> allreduce g -> ||Zg||^2 -> allreduce
//                   -> tau_d -> update + ball projection
//   csc_objective   dense residual r'' (refreshes the cache) + ||z||_1 -> allreduce -> F
// NCCL (world > 1) is loaded with dlopen("libnccl.so.2") at csc_init; single-GPU
// contexts never touch it.
#include "../../include/csc.h"
#include "csc_internal.cuh"

#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

using csc::Geom;

namespace {

std::mutex g_err_mu;
std::string g_init_err;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  bool load(std::string* err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      *err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return false;
    }
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(dlsym(h, "ncclAllReduce"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    CommGetAsyncError = reinterpret_cast<decltype(CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    if (!GetUniqueId || !CommInitRank || !CommDestroy || !AllReduce || !GetErrorString) {
      *err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

constexpr double kBcdRidge = 1e-10;  // DESIGN.md reading B2

// device scalar slots
// kCounter: a block counter of the fused fixup reductions (zero, cleared by each launch); kCnt:
// csc_count_nonzero (host mirror only)
enum DSlot { kSqR = 0, kL1 = 1, kZg2 = 2, kGG = 3, kLhat = 4, kCounter = 6, kCnt = 7, kNumD = 8 };
enum FSlot { kTauZ = 0, kTauD = 1, kNumF = 4 };
constexpr size_t kScalBytes = sizeof(double) * kNumD + sizeof(float) * kNumF;  // dscal then fscal, one block

}  // namespace

struct csc_ctx {
  Geom g{};
  int world = 1, rank = 0, device = 0;
  cudaStream_t st = nullptr;
  // scratch
  float* r = nullptr;          // [N][H][W] residual cache
  float* part = nullptr;       // conv k-split partials
  int ksplit = 1;              // dense-pass k split
  double* sq_part = nullptr;   // per-block partials
  double* l1_part = nullptr;
  int part_cap = 0;
  double* gpart = nullptr;     // [G][K][S*S]
  int G = 1;
  double* gsum = nullptr;      // [K][S*S]
  float* g32 = nullptr;
  uint32_t* colw = nullptr;    // mask column words
  double* lip_part = nullptr;
  double* dscal = nullptr;
  float* fscal = nullptr;
  double* h_dscal = nullptr;   // pinned host mirrors
  float* h_fscal = nullptr;
  // pipelined iterations (csc_iterate_staged_async): a ring of 2 pinned result slots and their events
  double* h_res_d[2] = {nullptr, nullptr};
  float* h_res_f[2] = {nullptr, nullptr};
  cudaEvent_t res_ev[2] = {nullptr, nullptr};
  float res_lam[2] = {0.f, 0.f};
  int res_pending = -1;  // slot of the enqueued iteration whose results were not returned yet
  int res_next = 0;
  // residual cache
  bool cache_valid = false;
  // L_D(d) and tau_z = 1/L_D of the filters last used (d changes only through the filter steps, which
  // clear it, or outside the API, which requires csc_invalidate): one bound per filter update, not per
  // code step (config 4 runs 10 code steps per filter step)
  bool lip_valid = false;
  const float* lip_d = nullptr;
  const float* cx = nullptr;
  const float* cd = nullptr;
  const float* cz = nullptr;
  // tensor-core dense path (csc_tc.cu)
  bool tc_on = false;
  csc::TcPlan tc{};
  float* tc_part = nullptr;
  int* tc_sched = nullptr;  // conv_h: the balanced item schedule (c->tc.sched points here)
  int* ct_sched = nullptr;  // code_h: the balanced item schedule (c->ct.sched points here)
  float* tc_bimg = nullptr;
  // fp16-split dense pass: scale bounds (float bits): [0] = bound of max|z|, [1] = max|filter|
  uint32_t* smax = nullptr;
  bool zmax_known = false;
  const float* zmax_ptr = nullptr;
  // tensor-core filter gradient (csc_wgrad_tc.cu)
  bool wg_tc_on = false;
  csc::WgTcPlan wg{};
  // fp16-rate filter gradient (csc_wgrad_h.cu): needs the max|z| bound of the fp16 dense path
  bool wh_on = false;
  csc::WhPlan wh{};
  uint32_t* wmax = nullptr;    // max|r'| (float bits) for the fp16-split filter gradient
  // tensor-core dense-then-mask code step (csc_code_tc.cu)
  bool ct_on = false;
  csc::CodeTcPlan ct{};
  uint32_t* mwords = nullptr;  // selection-word mask [wper*nkg][Hc*Wc]
  float* a3_part = nullptr;    // a3' band partials of the fp16-split code step [nkg][N][nbands][BR+P][W]
  csc::TmapCache tm_code[2];   // code step: z, selection words
  csc::TmapCache tm_adm[2];    // ADMM's D^T e pass through the code-step kernel (plain mode)
  csc::TmapCache tm_conv;      // dense pass: z
  csc::TmapCache tm_conv_adm;  // dense pass over the ADMM expansion buffer
  csc::TmapCache tm_wgrad;     // filter gradient: z
  uint32_t* rmax = nullptr;    // max|r| (float bits) for the fp16-split code step
  int step_rule = CSC_STEP_LIPSCHITZ;  // built-in tau_z rule (csc_set_step_rule)
  // projected block-coordinate filter update scratch (csc_bcd.cu), allocated on first use
  double* bcd_gpart = nullptr;  // [K][splits][M][M]
  double* bcd_ainv = nullptr;   // [K][M][M]
  uint8_t* bcd_flags = nullptr; // [K]
  double* bcd_part = nullptr;   // [gk blocks][M]
  double* bcd_vec = nullptr;    // gk[M], dl[M]
  double* bcd_gq = nullptr;     // lag-structured Gram prefix sums
  double* bcd_cfull = nullptr;  // [K][M][M]
  // online surrogates (Eq.7), allocated by the first csc_surrogate_reset / update
  double* sur_C = nullptr;      // [K][K][M][M]
  double* sur_B = nullptr;      // [K][M]
  double* sur_pp = nullptr;     // batch Gram partials
  double* sur_diag = nullptr;   // [K][M][M]
  int64_t sur_t = 0;
  bool last_eso = false;       // the last code step used per-filter taus
  int mask_mode = CSC_MASK_ENTRY;  // csc_set_mask_mode
  const uint32_t* iter_off = nullptr;  // csc_set_iter_offset: device-side mask-iteration offset
  // double-buffered image staging (csc_stage_images / csc_iterate_staged)
  cudaStream_t cp_st = nullptr;
  float* stage[2] = {nullptr, nullptr};
  cudaEvent_t st_ready[2] = {nullptr, nullptr};
  cudaEvent_t st_free[2] = {nullptr, nullptr};
  bool staged[2] = {false, false};
  bool st_used[2] = {false, false};
  float* tauk = nullptr;       // [K] per-filter tau_z of the ESO rule
  // ADMM code solver scratch (csc_admm.cu), allocated by the first csc_code_step_admm
  float* adm_zd = nullptr;      // [N][K][Hc][Wc] scatter target of the operator (0 off the mask)
  float* adm_e = nullptr;       // [N][H][W] operator output
  float* adm_cd = nullptr;      // [N][K][Hc][Wc] dense D^T e of the tensor-core correlation
  uint32_t* adm_bits = nullptr; // canonical mask bits
  uint32_t* adm_idx = nullptr;  // selected positions [K*Hc*Wc]
  uint32_t* adm_woff = nullptr; // set bits before each mask word
  uint32_t* adm_cnt = nullptr;
  uint64_t* adm_off = nullptr;
  uint64_t* adm_row = nullptr;  // row offsets [K*Hc + 1]
  uint64_t* adm_mc = nullptr;   // device count + pinned host mirror
  uint64_t* h_adm_mc = nullptr;
  uint32_t* adm_bound = nullptr;
  double* adm_part = nullptr;   // [2][N][blocks]
  double* adm_s = nullptr;      // per-image CG scalars [2][N]
  float* adm_vec = nullptr;     // 7 compact vectors W Y U R PV Q ATB [N][cap]
  int64_t adm_cap = 0;
  ncclComm_t comm = nullptr;
  bool nvtx = false;  // csc_set_nvtx / CSC_NVTX=1
  double* gf_scratch = nullptr;  // grad_finish block sums + counter
  uint64_t* cnt_dev = nullptr;  // csc_count_nonzero
  uint64_t launches = 0;
  std::string err;
  // profiling
  struct Rec { cudaEvent_t a, b; int cls; };
  bool prof_on = false;
  uint32_t prof_mask = 0xFFFFFFFFu;  // kernel classes timed while prof_on (csc_profile_set_classes)
  bool sampled = false;              // csc_profile_sample accumulated the pending pairs (keep them)
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  std::vector<cudaEvent_t> retired;  // events of sampled (graph-captured) pairs, destroyed with the context
  double prof_ms[CSC_K_NCLASS] = {0};
  uint64_t prof_n[CSC_K_NCLASS] = {0};
};

namespace {

// NVTX range around one entry point (csc_set_nvtx); header-only NVTX v3, inert without a tool
struct NvtxScope {
  bool on;
  NvtxScope(const csc_ctx* c, const char* name) : on(c != nullptr && c->nvtx) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxScope() {
    if (on) nvtxRangePop();
  }
};

csc_status fail(csc_ctx* c, csc_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

#define CSC_CUDA(ctx, call)                                                                      \
  do {                                                                                           \
    cudaError_t _e = (call);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      return fail((ctx), CSC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));      \
  } while (0)

cudaEvent_t prof_event(csc_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// A profiling event on the context stream; under stream capture it becomes an external event-record node
// of the graph (re-recorded by every replay, csc_profile_sample)
void prof_record(csc_ctx* c, cudaEvent_t e) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, c->st, cudaEventRecordExternal);
  else cudaEventRecord(e, c->st);
}

// Launch `call` (nk kernels of class cls); with profiling on, bracket it with events.
#define CSC_LAUNCH_C(ctx, cls, nk, call)                                                         \
  do {                                                                                           \
    cudaEvent_t _ea = nullptr, _eb = nullptr;                                                    \
    const bool _pr = (ctx)->prof_on && (((ctx)->prof_mask >> (cls)) & 1u);                       \
    if (_pr) {                                                                                   \
      _ea = prof_event(ctx);                                                                     \
      _eb = prof_event(ctx);                                                                     \
      prof_record(ctx, _ea);                                                                     \
    }                                                                                            \
    cudaError_t _e = (call);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      return fail((ctx), CSC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));      \
    if (_pr) {                                                                                   \
      prof_record(ctx, _eb);                                                                     \
      (ctx)->pending.push_back({_ea, _eb, (cls)});                                               \
    }                                                                                            \
    (ctx)->launches += (nk);                                                                     \
  } while (0)
#define CSC_LAUNCH(ctx, nk, call) CSC_LAUNCH_C(ctx, CSC_K_SMALL, nk, call)

#define CSC_NCCL(ctx, call)                                                                      \
  do {                                                                                           \
    ncclResult_t _r = (call);                                                                    \
    if (_r != ncclSuccess)                                                                       \
      return fail((ctx), CSC_ERR_NCCL, std::string(#call) + ": " + g_nccl.GetErrorString(_r));   \
  } while (0)

bool aligned4(const void* p) { return p != nullptr && (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

int64_t n_pix(const Geom& g) { return static_cast<int64_t>(g.N) * g.H * g.W; }

csc_status allreduce_d(csc_ctx* c, double* buf, size_t count) {
  if (c->world <= 1) return CSC_OK;
  CSC_NCCL(c, g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->st));
  return CSC_OK;
}

// Tensor-core dense pass y = sum_k f_k * z_k into the band partials (TMA-fed SS kernel when the
// plan says so, else the TMEM-fed kernel).
// The fp16 split needs a bound of max|z|: exact after csc_zero_codes or an absmax pass, then raised by
// every code step (T6).
cudaError_t ensure_zmax(csc_ctx* c, const float* z) {
  if (!c->zmax_known || c->zmax_ptr != z) {
    cudaError_t e = csc::launch_absmax(z, static_cast<int64_t>(c->g.N) * c->g.K * c->g.Hc * c->g.Wc, c->smax, c->st);
    if (e != cudaSuccess) return e;
    c->launches += 1;
    c->zmax_known = true;
    c->zmax_ptr = z;
  }
  return cudaSuccess;
}

cudaError_t conv_tc_any(csc_ctx* c, const float* z, const float* filt, double* l1p, bool precise = false) {
  if (c->tc.half) {
    cudaError_t ez = ensure_zmax(c, z);
    if (ez != cudaSuccess) return ez;
    return csc::launch_conv_h(c->g, c->tc, &c->tm_conv, z, filt, c->tc_bimg, c->smax, c->smax + 1, c->tc_part, l1p,
                              c->st, true, precise);
  }
  if (c->tc.ss) {
    cudaError_t e = csc::launch_tc_bimg(c->g, c->tc, filt, c->tc_bimg, c->st);
    if (e != cudaSuccess) return e;
    return csc::launch_conv_ss(c->g, c->tc, &c->tm_conv, z, c->tc_bimg, c->tc_part, l1p, c->st);
  }
  return csc::launch_conv_tc(c->g, c->tc, z, filt, c->tc_bimg, c->tc_part, l1p, c->st);
}

// Dense residual pass r = Dz - x, plus sum r^2 -> dscal[kSqR] and (optional)
// ||z||_1 -> dscal[kL1]; both local to this rank.
csc_status dense_residual(csc_ctx* c, const float* x, const float* d, const float* z, bool want_l1) {
  const Geom& g = c->g;
  int nb = 0;
  double* l1p = want_l1 ? c->l1_part : nullptr;
  if (g.N == 0) {
    CSC_CUDA(c, cudaMemsetAsync(c->dscal, 0, sizeof(double) * 2, c->st));
    return CSC_OK;
  }
  if (c->tc_on) {
    CSC_LAUNCH_C(c, CSC_K_CONV, 1 + c->tc.nks, conv_tc_any(c, z, d, l1p));
    csc::FixupSums fs;
    fs.out_sq = c->dscal + kSqR;
    if (want_l1) {
      fs.l1_part = c->l1_part;
      fs.nl1 = c->tc.nks * c->tc.grid;
      fs.out_l1 = c->dscal + kL1;
    }
    fs.counter = reinterpret_cast<unsigned long long*>(c->dscal + kCounter);
    CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1,
                 csc::launch_conv_tc_fixup(g, c->tc, c->tc_part, x, c->r, csc::kConvResidual, c->sq_part, c->st, &fs));
    c->cache_valid = true;
    c->cx = x;
    c->cd = d;
    c->cz = z;
    return CSC_OK;
  }
  CSC_LAUNCH_C(c, CSC_K_CONV, 1, csc::launch_conv_fwd(g, z, d, x, c->r, c->part, c->ksplit, csc::kConvResidual, c->sq_part, l1p,
                                        c->st, &nb));
  if (c->ksplit == 1) {
    CSC_LAUNCH(c, 1, csc::launch_reduce_sum(c->sq_part, nb, c->dscal + kSqR, 1.0, c->st));
  } else {
    CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1, csc::launch_conv_finalize(g, c->part, c->ksplit, x, c->r, csc::kConvResidual, c->sq_part, c->st));
    CSC_LAUNCH(c, 1, csc::launch_reduce_sum(c->sq_part, csc::kFinalizeBlocks, c->dscal + kSqR, 1.0, c->st));
  }
  if (want_l1) CSC_LAUNCH(c, 1, csc::launch_reduce_sum(c->l1_part, nb, c->dscal + kL1, 1.0, c->st));
  c->cache_valid = true;
  c->cx = x;
  c->cd = d;
  c->cz = z;
  return CSC_OK;
}

// The code step raises the max|z| bound of the fp16-split dense pass when it writes the tracked z.
uint32_t* zbound(csc_ctx* c, const float* z) {
  if (c->smax == nullptr) return nullptr;
  if (c->zmax_ptr != z) c->zmax_known = false;
  return c->zmax_known ? c->smax : nullptr;
}

// out = D v - x (plain D v when x == nullptr) for a code-shaped v: the dense pass of
// dense_residual into a caller buffer, without touching the residual cache.
csc_status dense_apply(csc_ctx* c, const float* x, const float* d, const float* v, float* out) {
  const Geom& g = c->g;
  if (c->tc_on) {
    CSC_LAUNCH_C(c, CSC_K_CONV, 1 + c->tc.nks, conv_tc_any(c, v, d, nullptr));
    CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1,
                 csc::launch_conv_tc_fixup(g, c->tc, c->tc_part, x, out, csc::kConvResidual, c->sq_part, c->st));
    return CSC_OK;
  }
  int nb = 0;
  CSC_LAUNCH_C(c, CSC_K_CONV, 1, csc::launch_conv_fwd(g, v, d, x, out, c->part, c->ksplit, csc::kConvResidual,
                                                      c->sq_part, nullptr, c->st, &nb));
  if (c->ksplit > 1)
    CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1,
                 csc::launch_conv_finalize(g, c->part, c->ksplit, x, out, csc::kConvResidual, c->sq_part, c->st));
  return CSC_OK;
}

// scratch of the block-coordinate filter updates (csc_filter_step_bcd, csc_filter_step_surrogate)
bool bcd_scratch(csc_ctx* c) {
  if (c->bcd_gpart != nullptr) return true;
  const Geom& g = c->g;
  const int M = g.S * g.S;
  const int ns = csc::bcd_gram_splits(g);
  const int nb = csc::bcd_gk_blocks(g);
  auto al = [](void** q, size_t bytes) { return cudaMalloc(q, bytes < 16 ? 16 : bytes) == cudaSuccess; };
  bool ok = al(reinterpret_cast<void**>(&c->bcd_gpart), sizeof(double) * g.K * ns * M * M);
  ok = ok && al(reinterpret_cast<void**>(&c->bcd_ainv), sizeof(double) * g.K * M * M);
  ok = ok && al(reinterpret_cast<void**>(&c->bcd_flags), static_cast<size_t>(g.K));
  ok = ok && al(reinterpret_cast<void**>(&c->bcd_part), sizeof(double) * (nb > 0 ? nb : 1) * M);
  ok = ok && al(reinterpret_cast<void**>(&c->bcd_vec), sizeof(double) * 2 * M);
  if (!ok) {
    cudaFree(c->bcd_gpart);
    c->bcd_gpart = nullptr;
    cudaGetLastError();
  }
  return ok;
}

bool cache_ok(const csc_ctx* c, const float* x, const float* d, const float* z) {
  return c->cache_valid && c->cx == x && c->cd == d && c->cz == z;
}

csc_status check_ptrs(csc_ctx* c, const void* x, const void* d, const void* z) {
  if (!c) return CSC_ERR_ARG;
  if (!aligned4(d)) return fail(c, CSC_ERR_ARG, "d must be a non-null 4-byte aligned device pointer");
  if (c->g.N > 0 && (!aligned4(x) || !aligned4(z)))
    return fail(c, CSC_ERR_ARG, "x and z must be non-null 4-byte aligned device pointers");
  return CSC_OK;
}

}  // namespace

extern "C" {

int csc_abi_version(void) { return CSC_ABI_VERSION; }

const char* csc_last_error(const csc_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_init_err.c_str();
}

uint64_t csc_launch_count(const csc_ctx* ctx) { return ctx ? ctx->launches : 0; }

uint32_t csc_kernel_variants(const csc_ctx* ctx) {
  if (!ctx) return 0;
  return (ctx->tc_on ? 1u : 0u) | (ctx->wg_tc_on ? 2u : 0u) | (ctx->ct_on ? 4u : 0u) |
         (ctx->tc_on && ctx->tc.ss ? 8u : 0u) | (ctx->tc_on && ctx->tc.half ? 16u : 0u) |
         (ctx->ct_on && ctx->ct.half ? 32u : 0u) | (ctx->wh_on && ctx->tc_on && ctx->tc.half ? 64u : 0u);
}

csc_status csc_nccl_unique_id(uint8_t out[128]) {
  if (!out) return CSC_ERR_ARG;
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  std::string err;
  if (!g_nccl.load(&err)) {
    std::lock_guard<std::mutex> lk2(g_err_mu);
    g_init_err = err;
    return CSC_ERR_NCCL;
  }
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return CSC_ERR_NCCL;
  std::memcpy(out, id.internal, 128);
  return CSC_OK;
}

csc_status csc_init(const csc_dims* dims, csc_ctx** out) {
  auto init_fail = [](csc_status s, const std::string& m) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    g_init_err = m;
    return s;
  };
  if (!dims || !out) return init_fail(CSC_ERR_ARG, "null dims/out");
  const csc_dims& D = *dims;
  if (D.K < 1 || D.n_local < 0 || D.s < 1 || (D.s % 2) == 0 || D.H < D.s || D.W < D.s)
    return init_fail(CSC_ERR_ARG, "invalid dims: need K>=1, n_local>=0, odd s>=1, H,W>=s");
  if (!(D.world == 1 || D.world == 2 || D.world == 4 || D.world == 8) || D.rank < 0 || D.rank >= D.world)
    return init_fail(CSC_ERR_ARG, "world must be 1,2,4,8 and 0<=rank<world");
  if (D.world > 1 && D.nccl_id == nullptr) return init_fail(CSC_ERR_ARG, "nccl_id required for world>1");
  if (!csc::filter_size_supported(D.s)) return init_fail(CSC_ERR_SHAPE, "filter size s not compiled (1,3,5,7,9,11)");
  if (static_cast<int64_t>(D.H + D.s - 1) * (D.W + D.s - 1) * D.K > (int64_t(1) << 31))
    return init_fail(CSC_ERR_SHAPE, "K*(H+s-1)*(W+s-1) exceeds 2^31 per image");

  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return init_fail(CSC_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(ce));
  if (D.device < 0 || D.device >= ndev) return init_fail(CSC_ERR_ARG, "device ordinal out of range");
  ce = cudaSetDevice(D.device);
  if (ce != cudaSuccess) return init_fail(CSC_ERR_CUDA, cudaGetErrorString(ce));
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, D.device);
  if (prop.major != 10)
    return init_fail(CSC_ERR_CUDA, "kernels are compiled for sm_100a only (B200); found sm_" +
                                       std::to_string(prop.major) + std::to_string(prop.minor));

  csc_ctx* c = new csc_ctx();
  c->g.N = D.n_local;
  c->g.K = D.K;
  c->g.S = D.s;
  c->g.H = D.H;
  c->g.W = D.W;
  c->g.Hc = D.H + D.s - 1;
  c->g.Wc = D.W + D.s - 1;
  c->g.P = D.s - 1;
  c->world = D.world;
  c->rank = D.rank;
  c->device = D.device;
  c->st = static_cast<cudaStream_t>(D.stream);
  const Geom& g = c->g;

  // dense-pass k split: aim for >= ~8 CTAs per SM over the grid
  const int tiles = csc::ceil_div(g.W, csc::kConvTW) * csc::ceil_div(g.H, csc::kConvTH) * (g.N > 0 ? g.N : 1);
  int ks = csc::ceil_div(prop.multiProcessorCount * 8, tiles);
  if (ks > g.K) ks = g.K;
  if (ks > 32) ks = 32;
  if (ks < 1) ks = 1;
  c->ksplit = ks;
  // filter-gradient tile groups
  const int wtiles = csc::ceil_div(g.W, csc::kWgTW) * csc::ceil_div(g.H, csc::kWgTH) * (g.N > 0 ? g.N : 1);
  int G = csc::ceil_div(prop.multiProcessorCount * 8, g.K);
  if (G > wtiles) G = wtiles;
  if (G < 1) G = 1;
  c->G = G;

  const int64_t npix = n_pix(g);
  const int M = g.S * g.S;
  const int NB = csc::ceil_div(g.Hc, 32);
  int cap = csc::conv_fwd_blocks(g, ks);
  if (cap < csc::kFinalizeBlocks) cap = csc::kFinalizeBlocks;
  c->part_cap = cap;
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (bytes == 0) bytes = 16;
    return cudaMalloc(p, bytes) == cudaSuccess;
  };
  bool ok = true;
  ok = ok && alloc(reinterpret_cast<void**>(&c->r), sizeof(float) * npix);
  if (ks > 1) ok = ok && alloc(reinterpret_cast<void**>(&c->part), sizeof(float) * npix * ks);
  ok = ok && alloc(reinterpret_cast<void**>(&c->sq_part), sizeof(double) * cap);
  ok = ok && alloc(reinterpret_cast<void**>(&c->l1_part), sizeof(double) * cap);
  // tensor-core filter gradient unless CSC_WGRAD_PATH=simt (needs Hc*Wc % 4 == 0 for the TMA view of z)
  {
    const char* nv = std::getenv("CSC_NVTX");
    c->nvtx = nv != nullptr && std::atoi(nv) != 0;
  }
  {
    const char* ev = std::getenv("CSC_WGRAD_PATH");
    const bool force_simt = ev != nullptr && std::string(ev) == "simt";
    const bool force_tf32 = ev != nullptr && std::string(ev) == "tf32";
    if (!force_simt && csc::wgrad_tc_supported(g)) {
      c->wg = csc::wgrad_tc_plan(g, prop.multiProcessorCount);
      c->wg_tc_on = true;
    }
    if (!force_simt && !force_tf32 && csc::wgrad_h_supported(g)) {
      c->wh = csc::wgrad_h_plan(g, prop.multiProcessorCount);
      c->wh_on = c->wh.ok;
      if (c->wh_on) ok = ok && alloc(reinterpret_cast<void**>(&c->wmax), sizeof(uint32_t) * 2);
    }
  }
  // tensor-core code step unless CSC_CODE_PATH=simt
  {
    const char* ev = std::getenv("CSC_CODE_PATH");
    const bool force_simt = ev != nullptr && std::string(ev) == "simt";
    const bool force_tc = ev != nullptr && std::string(ev) == "tc";
    if (!force_simt && !force_tc && csc::code_h_supported(g)) {
      c->ct = csc::code_h_plan(g, prop.multiProcessorCount);
      if (!c->ct.ok) c->ct = csc::code_tc_plan(g, prop.multiProcessorCount);
    } else if (!force_simt && csc::code_tc_supported(g)) {
      c->ct = csc::code_tc_plan(g, prop.multiProcessorCount);
    }
    if (!force_simt && (csc::code_h_supported(g) || csc::code_tc_supported(g))) {
      if (c->ct.ok) {
        c->ct_on = true;
        ok = ok && alloc(reinterpret_cast<void**>(&c->mwords), sizeof(uint32_t) * c->ct.sw_words);
        if (c->ct.half) ok = ok && alloc(reinterpret_cast<void**>(&c->a3_part), sizeof(float) * c->ct.a3_floats);
        if (ok && c->ct.half) {
          std::vector<int> sched;
          csc::code_h_schedule(g, c->ct, sched);
          ok = alloc(reinterpret_cast<void**>(&c->ct_sched), sizeof(int) * sched.size()) &&
               cudaMemcpy(c->ct_sched, sched.data(), sizeof(int) * sched.size(), cudaMemcpyHostToDevice) == cudaSuccess;
          c->ct.sched = c->ct_sched;
        }
        ok = ok && alloc(reinterpret_cast<void**>(&c->rmax), sizeof(uint32_t) * 4);
      }
    }
  }
  int gpart_groups = c->wg_tc_on && c->wg.G > G ? c->wg.G : G;
  if (c->wh_on && c->wh.G > gpart_groups) gpart_groups = c->wh.G;
  ok = ok && alloc(reinterpret_cast<void**>(&c->gpart), sizeof(double) * static_cast<size_t>(gpart_groups) * g.K * M);
  ok = ok && alloc(reinterpret_cast<void**>(&c->gsum), sizeof(double) * g.K * M);
  ok = ok && alloc(reinterpret_cast<void**>(&c->g32), sizeof(float) * g.K * M);
  ok = ok && alloc(reinterpret_cast<void**>(&c->tauk), sizeof(float) * g.K);
  ok = ok && alloc(reinterpret_cast<void**>(&c->colw), sizeof(uint32_t) * static_cast<size_t>(g.K) * NB * g.Wc);
  ok = ok && alloc(reinterpret_cast<void**>(&c->lip_part), sizeof(double) * (64 * 64 * csc::ceil_div(g.K, 2) + 64));
  // the fp64 and fp32 scalars share one block (fscal follows dscal): one D2H copy reads both
  ok = ok && alloc(reinterpret_cast<void**>(&c->dscal), kScalBytes);
  if (ok) c->fscal = reinterpret_cast<float*>(c->dscal + kNumD);
  ok = ok && alloc(reinterpret_cast<void**>(&c->gf_scratch), sizeof(double) * (csc::ceil_div(g.K * g.S * g.S, 256) + 1));
  ok = ok && cudaMallocHost(reinterpret_cast<void**>(&c->h_dscal), kScalBytes) == cudaSuccess;
  if (ok) c->h_fscal = reinterpret_cast<float*>(c->h_dscal + kNumD);
  // tensor-core dense path unless CSC_DENSE_PATH=simt
  {
    const char* ev = std::getenv("CSC_DENSE_PATH");
    const bool force_simt = ev != nullptr && std::string(ev) == "simt";
    if (!force_simt && g.N > 0 && csc::conv_tc_supported(g)) {
      const char* ev2 = std::getenv("CSC_CONV_PATH");
      const bool force_tmem = ev2 != nullptr && std::string(ev2) == "tmem";
      const bool force_ss = ev2 != nullptr && std::string(ev2) == "ss";
      bool planned = false;
      if (!force_tmem && !force_ss && csc::conv_h_supported(g)) planned = csc::conv_h_plan(g, prop.multiProcessorCount, c->tc);
      if (!planned && !force_tmem && csc::conv_ss_supported(g)) planned = csc::conv_ss_plan(g, prop.multiProcessorCount, c->tc);
      if (!planned) c->tc = csc::conv_tc_plan(g, prop.multiProcessorCount);
      c->tc_on = true;
      ok = ok && alloc(reinterpret_cast<void**>(&c->tc_part), sizeof(float) * c->tc.part_floats);
      if (ok && c->tc.half) {
        std::vector<int> sched;
        csc::conv_h_schedule(g, c->tc, sched);
        ok = alloc(reinterpret_cast<void**>(&c->tc_sched), sizeof(int) * sched.size()) &&
             cudaMemcpy(c->tc_sched, sched.data(), sizeof(int) * sched.size(), cudaMemcpyHostToDevice) == cudaSuccess;
        c->tc.sched = c->tc_sched;
      }
      ok = ok && alloc(reinterpret_cast<void**>(&c->tc_bimg), sizeof(float) * c->tc.bimg_floats);
      ok = ok && alloc(reinterpret_cast<void**>(&c->smax), sizeof(uint32_t) * 2);
      const int need = c->tc.nks * c->tc.grid;
      if (need > cap) {
        cudaFree(c->l1_part);
        c->l1_part = nullptr;
        ok = ok && alloc(reinterpret_cast<void**>(&c->l1_part), sizeof(double) * need);
      }
    }
  }
  if (!ok) {
    csc_destroy(c);
    return init_fail(CSC_ERR_OOM, "device allocation failed in csc_init");
  }
  cudaMemsetAsync(c->dscal, 0, sizeof(double) * kNumD, c->st);
  cudaMemsetAsync(c->gf_scratch, 0, sizeof(double) * (csc::ceil_div(g.K * g.S * g.S, 256) + 1), c->st);
  // the Lipschitz kernel's max / counter state past the partials starts at zero (launch_lipschitz)
  cudaMemsetAsync(c->lip_part, 0, sizeof(double) * (64 * 64 * csc::ceil_div(g.K, 2) + 64), c->st);
  cudaMemsetAsync(c->fscal, 0, sizeof(float) * kNumF, c->st);
  cudaMemsetAsync(c->gsum, 0, sizeof(double) * g.K * M, c->st);

  if (c->world > 1) {
    std::string err;
    {
      std::lock_guard<std::mutex> lk(g_nccl_mu);
      if (!g_nccl.load(&err)) {
        csc_destroy(c);
        return init_fail(CSC_ERR_NCCL, err);
      }
    }
    ncclUniqueId id;
    std::memcpy(id.internal, D.nccl_id, 128);
    ncclResult_t nr = g_nccl.CommInitRank(&c->comm, c->world, id, c->rank);
    if (nr != ncclSuccess) {
      const std::string m = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(nr);
      c->comm = nullptr;
      csc_destroy(c);
      return init_fail(CSC_ERR_NCCL, m);
    }
  }
  ce = cudaStreamSynchronize(c->st);
  if (ce != cudaSuccess) {
    csc_destroy(c);
    return init_fail(CSC_ERR_CUDA, cudaGetErrorString(ce));
  }
  *out = c;
  return CSC_OK;
}

csc_status csc_profile_enable(csc_ctx* c, int enable) {
  if (!c) return CSC_ERR_ARG;
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  for (auto& r : c->pending) {
    // sampled pairs may still be recorded by a captured graph: retire them instead of reusing them
    auto& dst = c->sampled ? c->retired : c->pool;
    dst.push_back(r.a);
    dst.push_back(r.b);
  }
  c->pending.clear();
  c->sampled = false;
  for (int i = 0; i < CSC_K_NCLASS; ++i) {
    c->prof_ms[i] = 0.0;
    c->prof_n[i] = 0;
  }
  c->prof_on = enable != 0;
  return CSC_OK;
}

csc_status csc_profile_sample(csc_ctx* c) {
  if (!c) return CSC_ERR_ARG;
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  for (auto& r : c->pending) {
    float ms = 0.f;
    CSC_CUDA(c, cudaEventElapsedTime(&ms, r.a, r.b));
    c->prof_ms[r.cls] += ms;
    c->prof_n[r.cls] += 1;
  }
  c->sampled = true;  // the pairs stay (a graph replays them); csc_profile_read then only reports
  return CSC_OK;
}

csc_status csc_profile_set_classes(csc_ctx* c, uint32_t class_mask) {
  if (!c) return CSC_ERR_ARG;
  c->prof_mask = class_mask;
  return CSC_OK;
}

csc_status csc_profile_read(csc_ctx* c, int cls, double* total_ms, uint64_t* launches) {
  if (!c || cls < 0 || cls >= CSC_K_NCLASS) return fail(c, CSC_ERR_ARG, "bad kernel class");
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  if (!c->sampled) {  // (csc_profile_sample already added the pairs it keeps)
    for (auto& r : c->pending) {
      float ms = 0.f;
      CSC_CUDA(c, cudaEventElapsedTime(&ms, r.a, r.b));
      c->prof_ms[r.cls] += ms;
      c->prof_n[r.cls] += 1;
      c->pool.push_back(r.a);
      c->pool.push_back(r.b);
    }
    c->pending.clear();
  }
  if (total_ms) *total_ms = c->prof_ms[cls];
  if (launches) *launches = c->prof_n[cls];
  return CSC_OK;
}

csc_status csc_destroy(csc_ctx* c) {
  if (!c) return CSC_OK;
  for (auto& r : c->pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto e : c->retired) cudaEventDestroy(e);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  cudaFree(c->r);
  cudaFree(c->part);
  cudaFree(c->sq_part);
  cudaFree(c->l1_part);
  cudaFree(c->gpart);
  cudaFree(c->gsum);
  cudaFree(c->cnt_dev);
  cudaFree(c->gf_scratch);
  cudaFree(c->g32);
  cudaFree(c->colw);
  cudaFree(c->mwords);
  cudaFree(c->a3_part);
  cudaFree(c->rmax);
  cudaFree(c->wmax);
  cudaFree(c->tauk);
  cudaFree(c->bcd_gpart);
  cudaFree(c->bcd_ainv);
  cudaFree(c->bcd_flags);
  cudaFree(c->bcd_part);
  cudaFree(c->bcd_vec);
  cudaFree(c->bcd_gq);
  cudaFree(c->bcd_cfull);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->stage[i]);
    if (c->st_ready[i]) cudaEventDestroy(c->st_ready[i]);
    if (c->st_free[i]) cudaEventDestroy(c->st_free[i]);
  }
  if (c->cp_st) cudaStreamDestroy(c->cp_st);
  cudaFree(c->sur_C);
  cudaFree(c->sur_B);
  cudaFree(c->sur_pp);
  cudaFree(c->sur_diag);
  cudaFree(c->adm_zd);
  cudaFree(c->adm_e);
  cudaFree(c->adm_cd);
  cudaFree(c->adm_bits);
  cudaFree(c->adm_idx);
  cudaFree(c->adm_woff);
  cudaFree(c->adm_cnt);
  cudaFree(c->adm_off);
  cudaFree(c->adm_mc);
  cudaFree(c->adm_row);
  cudaFreeHost(c->h_adm_mc);
  cudaFree(c->adm_bound);
  cudaFree(c->adm_part);
  cudaFree(c->adm_s);
  cudaFree(c->adm_vec);
  cudaFree(c->lip_part);
  cudaFree(c->tc_part);
  cudaFree(c->tc_sched);
  cudaFree(c->ct_sched);
  cudaFree(c->tc_bimg);
  cudaFree(c->smax);
  cudaFree(c->dscal);  // fscal, h_fscal and h_res_f point into the dscal / h_dscal / h_res_d blocks
  cudaFreeHost(c->h_dscal);
  for (int i = 0; i < 2; ++i) {
    cudaFreeHost(c->h_res_d[i]);
    if (c->res_ev[i]) cudaEventDestroy(c->res_ev[i]);
  }
  delete c;
  return CSC_OK;
}

csc_status csc_invalidate(csc_ctx* c) {
  if (!c) return CSC_ERR_ARG;
  c->cache_valid = false;
  c->zmax_known = false;
  c->lip_valid = false;
  return CSC_OK;
}

csc_status csc_zero_codes(csc_ctx* c, const float* x, float* z) {
  NvtxScope nvtx_scope(c, "csc_zero_codes");
  if (!c) return CSC_ERR_ARG;
  if (c->g.N > 0 && (!aligned4(x) || !aligned4(z))) return fail(c, CSC_ERR_ARG, "x, z must be device pointers");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  if (g.N > 0) {
    CSC_CUDA(c, cudaMemsetAsync(z, 0, sizeof(float) * static_cast<size_t>(g.N) * g.K * g.Hc * g.Wc, c->st));
    if (c->smax != nullptr) {
      CSC_CUDA(c, cudaMemsetAsync(c->smax, 0, sizeof(uint32_t), c->st));
      c->zmax_known = true;
      c->zmax_ptr = z;
    }
    CSC_LAUNCH(c, 1, csc::launch_neg_copy(x, c->r, n_pix(g), c->st));
  }
  c->cache_valid = true;
  c->cx = x;
  c->cz = z;
  c->cd = nullptr;  // r = -x holds for any d when z = 0
  return CSC_OK;
}

csc_status csc_code_step(csc_ctx* c, const float* x, const float* d, float* z, float lambda, float step_z,
                         double p, uint64_t seed, uint32_t iter, float* step_used) {
  NvtxScope nvtx_scope(c, "csc_code_step");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (!(lambda >= 0.f) || !std::isfinite(lambda)) return fail(c, CSC_ERR_ARG, "lambda must be finite and >= 0");
  if (!(step_z >= 0.f) || !std::isfinite(step_z)) return fail(c, CSC_ERR_ARG, "step_z must be finite and >= 0");
  if (!(p > 0.0 && p <= 1.0)) return fail(c, CSC_ERR_ARG, "p must be in (0, 1]");
  if (step_z == 0.f && c->step_rule == CSC_STEP_ESO && c->mask_mode == CSC_MASK_SECTOR8)
    return fail(c, CSC_ERR_ARG,
                "the ESO step (DESIGN.md E1) assumes independent per-code sampling; it is not valid for sector masks");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  // zero-code shortcut of csc_zero_codes: r = -x for any d
  const bool zero_ok = c->cache_valid && c->cd == nullptr && c->cx == x && c->cz == z;
  if (!zero_ok && !cache_ok(c, x, d, z)) {
    s = dense_residual(c, x, d, z, false);
    if (s != CSC_OK) return s;
  }
  const bool eso = step_z == 0.f && c->step_rule == CSC_STEP_ESO;
  if (step_z > 0.f) {
    CSC_LAUNCH(c, 1, csc::launch_set_f32(c->fscal + kTauZ, step_z, c->st));
    c->lip_valid = false;  // the tau_z slot now holds the explicit step
  } else {
    if (!(c->lip_valid && c->lip_d == d)) {
      CSC_LAUNCH_C(c, CSC_K_LIPSCHITZ, 2,
                   csc::launch_lipschitz(g, d, c->lip_part, c->dscal + kLhat, c->fscal + kTauZ, c->st));
      c->lip_valid = true;
      c->lip_d = d;
    }
    if (eso) CSC_LAUNCH(c, 1, csc::launch_eso_tau(g, d, p, c->dscal + kLhat, c->tauk, c->st));
  }
  c->last_eso = eso;
  // tau per filter (ESO) or one tau for all codes
  const float* tau_dev = eso ? c->tauk : c->fscal + kTauZ;
  const int tau_stride = eso ? 1 : 0;
  const uint64_t thr = static_cast<uint64_t>(std::floor(p * 4294967296.0));
  const int all_selected = thr >= (uint64_t(1) << 32) ? 1 : 0;
  bool a3_done = false;
  if (g.N > 0) {
    if (c->ct_on) {
      if (!all_selected)
        CSC_LAUNCH_C(c, CSC_K_MASK, 1, csc::launch_mask_selwords(g, c->ct, seed, iter, thr, c->mwords, c->st, c->mask_mode,
                                                                 c->iter_off));
      if (c->ct.half) {
        // masked step fused with the incremental residual r' = r + D dz (a3'): the cache then holds
        // D z_new - x for (x, d, z) and the filter step needs no dense residual pass
        CSC_LAUNCH(c, 1, csc::launch_absmax(c->r, n_pix(g), c->rmax, c->st));
        CSC_LAUNCH_C(c, CSC_K_CODE_STEP, 1,
                     csc::launch_code_h(g, c->ct, c->tm_code, c->r, d, z, all_selected ? nullptr : c->mwords, tau_dev,
                                        lambda, c->rmax, zbound(c, z), c->st, false, tau_stride, c->a3_part));
        CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1, csc::launch_code_a3_fixup(g, c->ct, c->a3_part, c->r, c->st));
        a3_done = true;
      } else {
        CSC_LAUNCH_C(c, CSC_K_CODE_STEP, 1,
                     csc::launch_code_tc(g, c->ct, c->r, d, z, all_selected ? nullptr : c->mwords, tau_dev,
                                         lambda, zbound(c, z), c->st, tau_stride));
      }
    } else {
      if (!all_selected)
        CSC_LAUNCH_C(c, CSC_K_MASK, 1, csc::launch_mask_colwords(g, seed, iter, thr, c->colw, c->st, c->mask_mode,
                                                                 c->iter_off));
      CSC_LAUNCH_C(c, CSC_K_CODE_STEP, 1, csc::launch_code_step(g, c->r, d, z, c->colw, all_selected, tau_dev, lambda,
                                                                zbound(c, z), c->st, tau_stride));
    }
  }
  if (a3_done || g.N == 0) {
    c->cache_valid = true;  // r' = r + D dz = D z_new - x  (a3')
    c->cx = x;
    c->cd = d;
    c->cz = z;
  } else {
    c->cache_valid = false;  // r no longer matches z
  }
  if (step_used) {
    CSC_CUDA(c, cudaMemcpyAsync(c->h_fscal + kTauZ, tau_dev, sizeof(float), cudaMemcpyDeviceToHost, c->st));
    CSC_CUDA(c, cudaStreamSynchronize(c->st));
    *step_used = c->h_fscal[kTauZ];
    if (!std::isfinite(*step_used)) return fail(c, CSC_ERR_NONFINITE, "tau_z is not finite");
  }
  return CSC_OK;
}

csc_status csc_set_step_rule(csc_ctx* c, int rule) {
  if (!c) return CSC_ERR_ARG;
  if (rule != CSC_STEP_LIPSCHITZ && rule != CSC_STEP_ESO) return fail(c, CSC_ERR_ARG, "unknown step rule");
  c->step_rule = rule;
  return CSC_OK;
}

csc_status csc_set_mask_mode(csc_ctx* c, int mode) {
  if (!c) return CSC_ERR_ARG;
  if (mode != CSC_MASK_ENTRY && mode != CSC_MASK_SECTOR8) return fail(c, CSC_ERR_ARG, "unknown mask mode");
  c->mask_mode = mode;
  return CSC_OK;
}

csc_status csc_set_iter_offset(csc_ctx* c, const uint32_t* offset_dev) {
  if (!c) return CSC_ERR_ARG;
  if (offset_dev != nullptr && !aligned4(offset_dev)) return fail(c, CSC_ERR_ARG, "offset_dev must be a device pointer");
  c->iter_off = offset_dev;
  return CSC_OK;
}

csc_status csc_read_step_z(csc_ctx* c, float* tau_dev) {
  if (!c || !aligned4(tau_dev)) return fail(c, CSC_ERR_ARG, "tau_dev must be a device pointer");
  CSC_CUDA(c, cudaSetDevice(c->device));
  if (c->last_eso) {
    CSC_CUDA(c, cudaMemcpyAsync(tau_dev, c->tauk, sizeof(float) * c->g.K, cudaMemcpyDeviceToDevice, c->st));
  } else {
    CSC_LAUNCH(c, 1, csc::launch_bcast_f32(tau_dev, c->fscal + kTauZ, c->g.K, c->st));
  }
  return CSC_OK;
}

csc_status csc_code_step_admm(csc_ctx* c, const float* x, const float* d, float* z, float lambda, float rho,
                              float alpha, int n_admm, int n_cg, double p, uint64_t seed, uint32_t iter) {
  NvtxScope nvtx_scope(c, "csc_code_step_admm");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (!(lambda > 0.f) || !std::isfinite(lambda)) return fail(c, CSC_ERR_ARG, "lambda must be finite and > 0");
  if (!(rho >= 0.f) || !std::isfinite(rho)) return fail(c, CSC_ERR_ARG, "rho must be finite and >= 0");
  if (!(alpha > 0.f && alpha < 2.f)) return fail(c, CSC_ERR_ARG, "alpha must be in (0, 2)");
  if (n_admm < 1 || n_cg < 1) return fail(c, CSC_ERR_ARG, "n_admm and n_cg must be >= 1");
  if (c->mask_mode != CSC_MASK_ENTRY) return fail(c, CSC_ERR_ARG, "the ADMM solver uses per-entry masks only");
  if (!(p > 0.0 && p <= 1.0)) return fail(c, CSC_ERR_ARG, "p must be in (0, 1]");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  if (g.N == 0) return CSC_OK;
  const int64_t nper = static_cast<int64_t>(g.K) * g.Hc * g.Wc;
  const int64_t ncode = static_cast<int64_t>(g.N) * nper;
  const int nbmax = std::max(csc::admm_blocks(g, (nper + 3) / 4 * 4), csc::admm_dtr_blocks(g));
  if (c->adm_zd == nullptr) {
    auto al = [](void** q, size_t bytes) { return cudaMalloc(q, bytes < 16 ? 16 : bytes) == cudaSuccess; };
    bool ok = al(reinterpret_cast<void**>(&c->adm_zd), sizeof(float) * ncode);
    ok = ok && al(reinterpret_cast<void**>(&c->adm_e), sizeof(float) * n_pix(g));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_bits), sizeof(uint32_t) * ((nper + 31) / 32));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_idx), sizeof(uint32_t) * nper);
    ok = ok && al(reinterpret_cast<void**>(&c->adm_woff), sizeof(uint32_t) * ((nper + 31) / 32));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_cnt), sizeof(uint32_t) * csc::admm_idx_blocks(g));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_off), sizeof(uint64_t) * csc::admm_idx_blocks(g));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_mc), sizeof(uint64_t));
    ok = ok && al(reinterpret_cast<void**>(&c->adm_row), sizeof(uint64_t) * (static_cast<int64_t>(g.K) * g.Hc + 1));
    ok = ok && cudaMallocHost(reinterpret_cast<void**>(&c->h_adm_mc), sizeof(uint64_t)) == cudaSuccess;
    ok = ok && al(reinterpret_cast<void**>(&c->adm_bound), sizeof(uint32_t) * 4);
    ok = ok && al(reinterpret_cast<void**>(&c->adm_part), sizeof(double) * 2 * g.N * nbmax);
    ok = ok && al(reinterpret_cast<void**>(&c->adm_s), sizeof(double) * 2 * g.N);
    if (!ok) {
      cudaGetLastError();
      return fail(c, CSC_ERR_OOM, "ADMM scratch allocation failed");
    }
  }
  // the selected positions of M^t (shared by every image), compacted; their count sizes the vectors
  const uint64_t thr = static_cast<uint64_t>(std::floor(p * 4294967296.0));
  CSC_LAUNCH_C(c, CSC_K_MASK, 1, csc::launch_mask_bits(g, seed, iter, thr, c->adm_bits, c->st));
  CSC_LAUNCH_C(c, CSC_K_ADMM, 3, csc::launch_admm_index(g, c->adm_bits, c->adm_cnt, c->adm_off, c->adm_mc,
                                                        c->adm_idx, c->adm_woff, c->st));
  CSC_CUDA(c, cudaMemcpyAsync(c->h_adm_mc, c->adm_mc, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  const int64_t mc = static_cast<int64_t>(*c->h_adm_mc);
  if (mc == 0) return CSC_OK;
  const int64_t ms = (mc + 3) / 4 * 4;
  if (ms > c->adm_cap) {
    cudaFree(c->adm_vec);
    c->adm_vec = nullptr;
    c->adm_cap = 0;
    int64_t cap = (ms + ms / 8 + 3) / 4 * 4;
    if (cap > (nper + 3) / 4 * 4) cap = (nper + 3) / 4 * 4;
    if (cudaMalloc(reinterpret_cast<void**>(&c->adm_vec), sizeof(float) * 7 * g.N * cap) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, CSC_ERR_OOM, "ADMM vector allocation failed");
    }
    c->adm_cap = cap;
  }
  CSC_LAUNCH_C(c, CSC_K_ADMM, 1, csc::launch_admm_row_off(g, c->adm_idx, mc, c->adm_row, c->st));
  // r = D z - x (the hot path's residual cache when it is valid)
  const bool zero_ok = c->cache_valid && c->cd == nullptr && c->cx == x && c->cz == z;
  if (!zero_ok && !cache_ok(c, x, d, z)) {
    s = dense_residual(c, x, d, z, false);
    if (s != CSC_OK) return s;
  }
  const int64_t cv = static_cast<int64_t>(g.N) * ms;
  float* W = c->adm_vec;
  float* Y = W + cv;
  float* U = Y + cv;
  float* R = U + cv;
  float* PV = R + cv;
  float* Q = PV + cv;
  float* ATB = Q + cv;  // explicit-residual mode only
  double* part_a = c->adm_part;  // <PV, Q> partials [N][admm_dtr_blocks] (masked_dtr blocks)
  double* part_b = part_a + static_cast<int64_t>(g.N) * nbmax;
  double* rr_cur = c->adm_s;
  double* rr_oth = rr_cur + g.N;
  const float rh = rho > 0.f ? rho : 10.f * lambda;
  const float kappa = lambda / rh;
  const int A = CSC_K_ADMM;
  bool first_conv = true;
  // A^T on the tensor cores (code_h in plain mode: dense D^T e, then a gather of the selected
  // codes) when the fp16-split code step is planned; else the SIMT masked gather-correlation.
  const char* dev = std::getenv("CSC_ADMM_DTR");
  const bool tc_dtr = c->ct_on && c->ct.half && !(dev != nullptr && std::string(dev) == "simt");
  if (tc_dtr && c->adm_cd == nullptr) {
    if (cudaMalloc(reinterpret_cast<void**>(&c->adm_cd), sizeof(float) * ncode) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, CSC_ERR_OOM, "ADMM correlation buffer allocation failed");
    }
  }
  const int nb_pq = tc_dtr ? csc::admm_blocks(g, ms) : csc::admm_dtr_blocks(g);
  float* E = c->adm_e;
  // all vectors (and their pads) start at 0: U = 0, and the pads stay 0 throughout
  CSC_CUDA(c, cudaMemsetAsync(c->adm_vec, 0, sizeof(float) * 7 * cv, c->st));
  // E = A v for the vector just expanded into Zd (max|v| in adm_bound[0] for the fp16 split)
  auto apply = [&]() -> csc_status {
    if (c->tc_on && c->tc.half) {
      CSC_LAUNCH_C(c, CSC_K_CONV, (first_conv ? 1 : 0) + c->tc.nks,
                   csc::launch_conv_h(g, c->tc, &c->tm_conv_adm, c->adm_zd, d, c->tc_bimg, c->adm_bound, c->smax + 1,
                                      c->tc_part, nullptr, c->st, first_conv, /*precise=*/true));
      CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1,
                   csc::launch_conv_tc_fixup(g, c->tc, c->tc_part, nullptr, E, csc::kConvResidual, c->sq_part, c->st));
      first_conv = false;
      return CSC_OK;
    }
    return dense_apply(c, nullptr, d, c->adm_zd, E);
  };
  // out = M D^T e (+ rho v and the <v, out> partials when v != null)
  auto dtr = [&](const float* e, const float* v, float* out, double* part, float sign) -> csc_status {
    if (tc_dtr) {
      CSC_LAUNCH(c, 1, csc::launch_absmax(e, n_pix(g), c->adm_bound + 1, c->st));
      CSC_LAUNCH_C(c, CSC_K_CODE_STEP, 1,
                   csc::launch_code_h(g, c->ct, c->tm_adm, e, d, c->adm_cd, nullptr, nullptr, 0.f, c->adm_bound + 1, nullptr,
                                      c->st, true));
      CSC_LAUNCH_C(c, CSC_K_ADMM, 1, csc::launch_admm_gather(g, c->adm_idx, mc, ms, c->adm_cd, v, rh, sign, out, part,
                                                             c->st));
      return CSC_OK;
    }
    CSC_LAUNCH_C(c, CSC_K_ADMM, 1, csc::launch_masked_dtr(g, c->adm_idx, c->adm_row, ms, e, d, v, rh, sign, out,
                                                          part, c->st));
    return CSC_OK;
  };
  CSC_LAUNCH_C(c, A, 1, csc::launch_admm_init(g, c->adm_idx, mc, ms, z, W, Y, c->st));
  // CG residual of the first right-hand side, R = ATB + rho (Y - U) - (A^T A + rho I) W with
  // W = Y = w0, U = 0:  R = A^T (b - A w0) = -M D^T r  (b - A w0 = x - D z = -r; A4)
  s = dtr(c->r, nullptr, R, nullptr, -1.f);
  if (s != CSC_OK) return s;
  CSC_LAUNCH_C(c, A, 2, csc::launch_sumsq(g, ms, R, part_b, rr_cur, c->st));
  // CSC_ADMM_RESID=explicit: recompute R = ATB + rho (Y - U) - (A^T A + rho I) W at every outer
  // iteration as the oracle does (one more operator application each), instead of carrying it.
  const char* rev = std::getenv("CSC_ADMM_RESID");
  const bool explicit_r = rev != nullptr && std::string(rev) == "explicit";
  auto q_of_w = [&]() -> csc_status {  // Q = (A^T A + rho I) W
    CSC_CUDA(c, cudaMemsetAsync(c->adm_bound, 0, sizeof(uint32_t), c->st));
    CSC_LAUNCH_C(c, A, 1, csc::launch_admm_expand(g, c->adm_bits, c->adm_woff, ms, W, nullptr, nullptr, nullptr,
                                                  c->adm_zd, c->adm_bound, c->st));
    csc_status s2 = apply();
    if (s2 != CSC_OK) return s2;
    return dtr(E, W, Q, nullptr, 1.f);
  };
  if (explicit_r) {
    s = q_of_w();
    if (s != CSC_OK) return s;
    CSC_LAUNCH_C(c, A, 2, csc::launch_cg_resid(g, ms, ATB, Y, U, Q, rh, R, part_b, rr_cur, true, c->st));
  }
  for (int it = 0; it < n_admm; ++it) {
    if (explicit_r && it > 0) {
      s = q_of_w();
      if (s != CSC_OK) return s;
      CSC_LAUNCH_C(c, A, 2, csc::launch_cg_resid(g, ms, ATB, Y, U, Q, rh, R, part_b, rr_cur, false, c->st));
    }
    for (int j = 0; j < n_cg; ++j) {
      // PV = R + (rr / rr_prev) PV  (PV = R first), expanded into Zd
      CSC_CUDA(c, cudaMemsetAsync(c->adm_bound, 0, sizeof(uint32_t), c->st));
      CSC_LAUNCH_C(c, A, 1, csc::launch_admm_expand(g, c->adm_bits, c->adm_woff, ms, R, PV, j == 0 ? nullptr : rr_oth,
                                                    rr_cur, c->adm_zd, c->adm_bound, c->st));
      s = apply();
      if (s != CSC_OK) return s;
      // Q = (A^T A + rho I) PV, part_a = <PV, Q>;  alpha_cg = rr / <PV,Q>;  W, R update; rr_new
      s = dtr(E, PV, Q, part_a, 1.f);
      if (s != CSC_OK) return s;
      CSC_LAUNCH_C(c, A, 2, csc::launch_cg_step(g, ms, rr_cur, part_a, nb_pq, W, R, PV, Q, part_b, rr_oth, c->st));
      std::swap(rr_cur, rr_oth);  // rr_cur = new |R|^2, rr_oth = previous
    }
    // y, u update; R carried to the next right-hand side, rr_cur = |R|^2
    CSC_LAUNCH_C(c, A, 2, csc::launch_admm_update(g, ms, W, Y, U, R, alpha, kappa, rh, part_b, rr_cur, c->st));
  }
  // z[M] = y; off-mask codes untouched.  The max|z| bound of the fp16 dense pass is raised.
  CSC_LAUNCH_C(c, A, 1, csc::launch_admm_scatter(g, c->adm_idx, mc, ms, Y, z, zbound(c, z), c->st));
  c->cache_valid = false;  // r no longer matches z
  return CSC_OK;
}

csc_status csc_filter_step_bcd(csc_ctx* c, const float* x, float* d, const float* z, int sweeps,
                               uint8_t* flags_out) {
  NvtxScope nvtx_scope(c, "csc_filter_step_bcd");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (sweeps < 1) return fail(c, CSC_ERR_ARG, "sweeps must be >= 1");
  if (c->g.S * c->g.S > 128) return fail(c, CSC_ERR_SHAPE, "block solve supports s*s <= 128");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  const int ns = csc::bcd_gram_splits(g);
  const int nb = csc::bcd_gk_blocks(g);
  if (!bcd_scratch(c)) return fail(c, CSC_ERR_OOM, "BCD scratch allocation failed");
  (void)nb;
  // r = D z - x (the residual cache when it is valid); the sweep keeps it current
  if (!cache_ok(c, x, d, z)) {
    s = dense_residual(c, x, d, z, false);
    if (s != CSC_OK) return s;
  }
  double* gk = c->bcd_vec;
  double* dl = c->bcd_vec + M;
  for (int sw = 0; sw < sweeps; ++sw) {
    // C_kk for all k on this rank's images, summed over ranks, then (C_kk + ridge)^-1.  Lag-structured
    // Gram (plane autocorrelation windows) when H, W > P unless CSC_BCD_GRAM=direct.
    const char* gev = std::getenv("CSC_BCD_GRAM");
    const bool lag = csc::bcd_lag_supported(g) && !(gev != nullptr && std::string(gev) == "direct");
    if (lag) {
      if (c->bcd_gq == nullptr) {
        if (cudaMalloc(reinterpret_cast<void**>(&c->bcd_gq), csc::bcd_lag_bytes(g)) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&c->bcd_cfull), sizeof(double) * g.K * M * M) != cudaSuccess) {
          cudaGetLastError();
          return fail(c, CSC_ERR_OOM, "BCD lag-Gram scratch allocation failed");
        }
      }
      CSC_LAUNCH_C(c, CSC_K_BCD, 2, csc::launch_bcd_lag_gram(g, z, c->bcd_gq, c->bcd_cfull, c->st));
      s = allreduce_d(c, c->bcd_cfull, static_cast<size_t>(g.K) * M * M);
      if (s != CSC_OK) return s;
      CSC_LAUNCH_C(c, CSC_K_BCD, 1, csc::launch_bcd_inverse_full(g, c->bcd_cfull, kBcdRidge, c->bcd_ainv,
                                                                 c->bcd_flags, c->st));
    } else {
      if (g.N > 0) {
        CSC_LAUNCH_C(c, CSC_K_BCD, 1, csc::launch_bcd_gram(g, z, c->bcd_gpart, c->st));
      } else {
        CSC_CUDA(c, cudaMemsetAsync(c->bcd_gpart, 0, sizeof(double) * g.K * ns * M * M, c->st));
      }
      s = allreduce_d(c, c->bcd_gpart, static_cast<size_t>(g.K) * ns * M * M);
      if (s != CSC_OK) return s;
      CSC_LAUNCH_C(c, CSC_K_BCD, 1, csc::launch_bcd_inverse(g, c->bcd_gpart, kBcdRidge, c->bcd_ainv, c->bcd_flags,
                                                            c->st));
    }
    for (int k = 0; k < g.K; ++k) {
      CSC_LAUNCH_C(c, CSC_K_BCD, nb > 0 ? 2 : 1, csc::launch_bcd_gk(g, k, z, c->r, c->bcd_part, gk, c->st));
      s = allreduce_d(c, gk, static_cast<size_t>(M));
      if (s != CSC_OK) return s;
      CSC_LAUNCH_C(c, CSC_K_BCD, g.N > 0 ? 2 : 1, csc::launch_bcd_update(g, k, gk, c->bcd_ainv, c->bcd_flags, d, dl, z,
                                                                         c->r, c->st));
    }
  }
  // the residual cache now belongs to the updated filters
  c->lip_valid = false;  // d changed
  c->cache_valid = true;
  c->cx = x;
  c->cd = d;
  c->cz = z;
  if (flags_out) {
    CSC_CUDA(c, cudaMemcpyAsync(flags_out, c->bcd_flags, static_cast<size_t>(g.K), cudaMemcpyDeviceToHost, c->st));
    CSC_CUDA(c, cudaStreamSynchronize(c->st));
  }
  return CSC_OK;
}

csc_status csc_surrogate_reset(csc_ctx* c) {
  if (!c) return CSC_ERR_ARG;
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  if (g.S * g.S > 128) return fail(c, CSC_ERR_SHAPE, "block solve supports s*s <= 128");
  if (c->sur_C == nullptr) {
    const int64_t np = static_cast<int64_t>(g.K) * (g.K + 1) / 2;
    auto al = [](void** q, size_t bytes) { return cudaMalloc(q, bytes < 16 ? 16 : bytes) == cudaSuccess; };
    bool ok = al(reinterpret_cast<void**>(&c->sur_C), sizeof(double) * g.K * g.K * M * M);
    ok = ok && al(reinterpret_cast<void**>(&c->sur_B), sizeof(double) * g.K * M);
    ok = ok && al(reinterpret_cast<void**>(&c->sur_pp), sizeof(double) * np * csc::sur_gram_splits(g) * M * M);
    ok = ok && al(reinterpret_cast<void**>(&c->sur_diag), sizeof(double) * g.K * M * M);
    if (!ok) {
      cudaFree(c->sur_C); cudaFree(c->sur_B); cudaFree(c->sur_pp); cudaFree(c->sur_diag);
      c->sur_C = c->sur_B = c->sur_pp = c->sur_diag = nullptr;
      cudaGetLastError();
      return fail(c, CSC_ERR_OOM, "surrogate allocation failed (K^2 M^2 doubles)");
    }
  }
  if (!bcd_scratch(c)) return fail(c, CSC_ERR_OOM, "BCD scratch allocation failed");
  CSC_CUDA(c, cudaMemsetAsync(c->sur_C, 0, sizeof(double) * g.K * g.K * M * M, c->st));
  CSC_CUDA(c, cudaMemsetAsync(c->sur_B, 0, sizeof(double) * g.K * M, c->st));
  c->sur_t = 0;
  return CSC_OK;
}

csc_status csc_surrogate_update(csc_ctx* c, const float* x, const float* z) {
  NvtxScope nvtx_scope(c, "csc_surrogate_update");
  if (!c) return CSC_ERR_ARG;
  if (c->g.N > 0 && (!aligned4(x) || !aligned4(z))) return fail(c, CSC_ERR_ARG, "x, z must be device pointers");
  if (c->sur_C == nullptr) {
    csc_status s0 = csc_surrogate_reset(c);
    if (s0 != CSC_OK) return s0;
  }
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  const int64_t t = c->sur_t + 1;
  // Eq.7 with the batch sums of all ranks: each rank folds (wo / world) C + wn (its batch) and the
  // all-reduce adds the ranks (C is identical on every rank)
  const double wo = static_cast<double>(t - 1) / static_cast<double>(t) / static_cast<double>(c->world);
  const double wn = 1.0 / static_cast<double>(t);
  // lag-structured pair Grams when H, W > P (CSC_BCD_GRAM=direct keeps the direct tap-pair sums)
  const char* gev = std::getenv("CSC_BCD_GRAM");
  const bool lag = csc::bcd_lag_supported(g) && g.N > 0 && !(gev != nullptr && std::string(gev) == "direct");
  CSC_LAUNCH_C(c, CSC_K_BCD, 1 + 3 * g.K + (lag ? 0 : 1),
               csc::launch_sur_update(g, x, z, lag ? nullptr : c->sur_pp, c->bcd_part, c->bcd_vec, wo, wn, c->sur_C,
                                      c->sur_B, c->st));
  csc_status s = allreduce_d(c, c->sur_C, static_cast<size_t>(g.K) * g.K * M * M);
  if (s != CSC_OK) return s;
  s = allreduce_d(c, c->sur_B, static_cast<size_t>(g.K) * M);
  if (s != CSC_OK) return s;
  c->sur_t = t;
  return CSC_OK;
}

csc_status csc_filter_step_surrogate(csc_ctx* c, float* d, int sweeps, uint8_t* flags_out) {
  NvtxScope nvtx_scope(c, "csc_filter_step_surrogate");
  if (!c || !aligned4(d)) return fail(c, CSC_ERR_ARG, "d must be a device pointer");
  if (sweeps < 1) return fail(c, CSC_ERR_ARG, "sweeps must be >= 1");
  if (c->sur_C == nullptr || c->sur_t < 1) return fail(c, CSC_ERR_ARG, "no surrogate: call csc_surrogate_update first");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  CSC_LAUNCH_C(c, CSC_K_BCD, 2, csc::launch_sur_prepare(g, c->sur_C, c->sur_diag, kBcdRidge, c->bcd_ainv,
                                                        c->bcd_flags, c->st));
  for (int sw = 0; sw < sweeps; ++sw)
    for (int k = 0; k < g.K; ++k)
      CSC_LAUNCH_C(c, CSC_K_BCD, 2, csc::launch_sur_filter(g, k, c->sur_C, c->sur_B, c->bcd_ainv, c->bcd_flags, d,
                                                           c->bcd_vec, c->bcd_vec + M, c->st));
  c->cache_valid = false;  // d changed
  c->lip_valid = false;
  if (flags_out) {
    CSC_CUDA(c, cudaMemcpyAsync(flags_out, c->bcd_flags, static_cast<size_t>(g.K), cudaMemcpyDeviceToHost, c->st));
    CSC_CUDA(c, cudaStreamSynchronize(c->st));
  }
  return CSC_OK;
}

csc_status csc_read_surrogate(csc_ctx* c, double* C_dev, double* B_dev, int64_t* t_out) {
  if (!c) return CSC_ERR_ARG;
  if (c->sur_C == nullptr) return fail(c, CSC_ERR_ARG, "no surrogate state");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  if (C_dev)
    CSC_CUDA(c, cudaMemcpyAsync(C_dev, c->sur_C, sizeof(double) * g.K * g.K * M * M, cudaMemcpyDeviceToDevice, c->st));
  if (B_dev) CSC_CUDA(c, cudaMemcpyAsync(B_dev, c->sur_B, sizeof(double) * g.K * M, cudaMemcpyDeviceToDevice, c->st));
  if (t_out) *t_out = c->sur_t;
  return CSC_OK;
}

// ||Z g||^2 of this rank's images for the fp32 copy g32 of the gradient -> dscal[kZg2] (no all-reduce):
// the precise dense pass (hi*hi and cross products in separate accumulators, reading T3)
static csc_status zg_pass(csc_ctx* c, const float* z) {
  const Geom& g = c->g;
  if (g.N > 0 && c->tc_on) {
    CSC_LAUNCH_C(c, CSC_K_CONV, 1 + c->tc.nks, conv_tc_any(c, z, c->g32, nullptr, true));
    csc::FixupSums fs;
    fs.out_sq = c->dscal + kZg2;
    fs.counter = reinterpret_cast<unsigned long long*>(c->dscal + kCounter);
    CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1,
                 csc::launch_conv_tc_fixup(g, c->tc, c->tc_part, nullptr, nullptr, csc::kConvSumSq, c->sq_part, c->st,
                                           &fs));
  } else if (g.N > 0) {
    int nb = 0;
    CSC_LAUNCH_C(c, CSC_K_CONV, 1, csc::launch_conv_fwd(g, z, c->g32, nullptr, nullptr, c->part, c->ksplit,
                                                        csc::kConvSumSq, c->sq_part, nullptr, c->st, &nb));
    if (c->ksplit == 1) {
      CSC_LAUNCH(c, 1, csc::launch_reduce_sum(c->sq_part, nb, c->dscal + kZg2, 1.0, c->st));
    } else {
      CSC_LAUNCH_C(c, CSC_K_CONV_FINALIZE, 1, csc::launch_conv_finalize(g, c->part, c->ksplit, nullptr, nullptr,
                                                                        csc::kConvSumSq, c->sq_part, c->st));
      CSC_LAUNCH(c, 1, csc::launch_reduce_sum(c->sq_part, csc::kFinalizeBlocks, c->dscal + kZg2, 1.0, c->st));
    }
  } else {
    CSC_CUDA(c, cudaMemsetAsync(c->dscal + kZg2, 0, sizeof(double), c->st));
  }
  return CSC_OK;
}

csc_status csc_filter_step(csc_ctx* c, const float* x, float* d, const float* z, float step_d, float* step_used) {
  NvtxScope nvtx_scope(c, "csc_filter_step");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (!(step_d >= 0.f) || !std::isfinite(step_d)) return fail(c, CSC_ERR_ARG, "step_d must be finite and >= 0");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  const int M = g.S * g.S;
  if (!cache_ok(c, x, d, z)) {
    s = dense_residual(c, x, d, z, false);
    if (s != CSC_OK) return s;
  }
  if (g.N > 0) {
    if (c->wh_on && c->tc_on && c->tc.half && (reinterpret_cast<uintptr_t>(z) & 15u) == 0) {
      // fp16-rate split: the bound of max|z| (as the dense pass) and max|r'|
      CSC_CUDA(c, ensure_zmax(c, z));
      CSC_LAUNCH(c, 1, csc::launch_absmax(c->r, n_pix(g), c->wmax, c->st));
      CSC_LAUNCH_C(c, CSC_K_WGRAD, 1,
                   csc::launch_wgrad_h(g, c->wh, &c->tm_wgrad, z, c->r, c->smax, c->wmax, c->gpart, c->st));
      CSC_LAUNCH(c, 1, csc::launch_wgrad_reduce(g, c->gpart, c->wh.G, c->gsum, c->st));
    } else if (c->wg_tc_on && (reinterpret_cast<uintptr_t>(z) & 15u) == 0) {
      CSC_LAUNCH_C(c, CSC_K_WGRAD, 1, csc::launch_wgrad_tc(g, c->wg, &c->tm_wgrad, z, c->r, c->gpart, c->st));
      CSC_LAUNCH(c, 1, csc::launch_wgrad_reduce(g, c->gpart, c->wg.G, c->gsum, c->st));
    } else {
      CSC_LAUNCH_C(c, CSC_K_WGRAD, 1, csc::launch_wgrad(g, z, c->r, c->G, c->gpart, c->st));
      CSC_LAUNCH(c, 1, csc::launch_wgrad_reduce(g, c->gpart, c->G, c->gsum, c->st));
    }
  } else {
    CSC_CUDA(c, cudaMemsetAsync(c->gsum, 0, sizeof(double) * g.K * M, c->st));
  }
  s = allreduce_d(c, c->gsum, static_cast<size_t>(g.K) * M);
  if (s != CSC_OK) return s;
  CSC_LAUNCH(c, 1, csc::launch_grad_finish(g, c->gsum, c->g32, c->dscal + kGG, c->gf_scratch, c->st));
  if (step_d == 0.f) {
    s = zg_pass(c, z);
    if (s != CSC_OK) return s;
    s = allreduce_d(c, c->dscal + kZg2, 1);
    if (s != CSC_OK) return s;
  }
  CSC_LAUNCH(c, 1, csc::launch_filter_tau(c->dscal + kGG, c->dscal + kZg2, step_d, c->fscal + kTauD, c->st));
  CSC_LAUNCH(c, 1, csc::launch_filter_update(g, d, c->gsum, c->fscal + kTauD, c->st));
  c->cache_valid = false;  // d changed
  c->lip_valid = false;
  if (step_used) {
    CSC_CUDA(c, cudaMemcpyAsync(c->h_fscal + kTauD, c->fscal + kTauD, sizeof(float), cudaMemcpyDeviceToHost, c->st));
    CSC_CUDA(c, cudaStreamSynchronize(c->st));
    *step_used = c->h_fscal[kTauD];
    if (!std::isfinite(*step_used)) return fail(c, CSC_ERR_NONFINITE, "tau_d is not finite");
  }
  return CSC_OK;
}

static csc_status objective_enqueue(csc_ctx* c, const float* x, const float* d, const float* z) {
  csc_status s = dense_residual(c, x, d, z, true);
  if (s != CSC_OK) return s;
  s = allreduce_d(c, c->dscal + kSqR, 2);
  if (s != CSC_OK) return s;
  CSC_CUDA(c, cudaMemcpyAsync(c->h_dscal, c->dscal, kScalBytes, cudaMemcpyDeviceToHost, c->st));
  return CSC_OK;
}

static csc_status objective_finish(csc_ctx* c, float lambda, double out[3]) {
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  const double half = 0.5 * c->h_dscal[kSqR];
  const double l1 = static_cast<double>(lambda) * c->h_dscal[kL1];
  out[0] = half + l1;
  out[1] = half;
  out[2] = l1;
  if (!std::isfinite(out[0])) return fail(c, CSC_ERR_NONFINITE, "objective is not finite");
  return CSC_OK;
}

csc_status csc_objective(csc_ctx* c, const float* x, const float* d, const float* z, float lambda, double out[3]) {
  NvtxScope nvtx_scope(c, "csc_objective");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (!out) return fail(c, CSC_ERR_ARG, "out must be a host pointer to 3 doubles");
  if (!(lambda >= 0.f) || !std::isfinite(lambda)) return fail(c, CSC_ERR_ARG, "lambda must be finite and >= 0");
  CSC_CUDA(c, cudaSetDevice(c->device));
  s = objective_enqueue(c, x, d, z);
  if (s != CSC_OK) return s;
  return objective_finish(c, lambda, out);
}

csc_status csc_objective_enqueue(csc_ctx* c, const float* x, const float* d, const float* z) {
  NvtxScope nvtx_scope(c, "csc_objective_enqueue");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  CSC_CUDA(c, cudaSetDevice(c->device));
  return objective_enqueue(c, x, d, z);
}

csc_status csc_objective_read(csc_ctx* c, float lambda, double out[3]) {
  if (!c || !out) return fail(c, CSC_ERR_ARG, "out must be a host pointer to 3 doubles");
  if (!(lambda >= 0.f) || !std::isfinite(lambda)) return fail(c, CSC_ERR_ARG, "lambda must be finite and >= 0");
  CSC_CUDA(c, cudaSetDevice(c->device));
  return objective_finish(c, lambda, out);
}

csc_status csc_stage_images(csc_ctx* c, const float* x_host, int slot) {
  if (!c || !x_host || slot < 0 || slot > 1) return fail(c, CSC_ERR_ARG, "x_host (host) and slot 0/1 required");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const size_t bytes = sizeof(float) * static_cast<size_t>(n_pix(c->g));
  if (c->cp_st == nullptr) {
    CSC_CUDA(c, cudaStreamCreateWithFlags(&c->cp_st, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CSC_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->stage[i]), bytes < 16 ? 16 : bytes));
      CSC_CUDA(c, cudaEventCreateWithFlags(&c->st_ready[i], cudaEventDisableTiming));
      CSC_CUDA(c, cudaEventCreateWithFlags(&c->st_free[i], cudaEventDisableTiming));
    }
  }
  if (c->st_used[slot]) CSC_CUDA(c, cudaStreamWaitEvent(c->cp_st, c->st_free[slot], 0));  // slot consumed
  if (bytes > 0) CSC_CUDA(c, cudaMemcpyAsync(c->stage[slot], x_host, bytes, cudaMemcpyHostToDevice, c->cp_st));
  CSC_CUDA(c, cudaEventRecord(c->st_ready[slot], c->cp_st));
  c->staged[slot] = true;
  return CSC_OK;
}

static csc_status iterate_impl(csc_ctx* c, const float* x_host, int slot, float* x, float* d, float* z, float lambda,
                               float step_z, float step_d, double p, uint64_t seed, uint32_t iter, double obj_out[3],
                               float taus_out[2]);

csc_status csc_load_staged(csc_ctx* c, int slot, float* x) {
  if (!c || slot < 0 || slot > 1 || c->stage[slot] == nullptr) return fail(c, CSC_ERR_ARG, "slot never staged");
  if (c->g.N > 0 && !aligned4(x)) return fail(c, CSC_ERR_ARG, "x must be a device pointer");
  CSC_CUDA(c, cudaSetDevice(c->device));
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CSC_CUDA(c, cudaStreamIsCapturing(c->st, &cs));
  const bool cap = cs == cudaStreamCaptureStatusActive;
  // inside a capture the events become external wait / record nodes: every replay waits for the slot's
  // latest copy and marks the slot free for csc_stage_images
  CSC_CUDA(c, cudaStreamWaitEvent(c->st, c->st_ready[slot], cap ? cudaEventWaitExternal : 0));
  const bool shift = c->cache_valid && c->cx == x && c->cz != nullptr;
  if (c->g.N > 0) CSC_LAUNCH(c, 1, csc::launch_stage_swap(c->stage[slot], x, c->r, n_pix(c->g), shift, c->st));
  CSC_CUDA(c, cudaEventRecordWithFlags(c->st_free[slot], c->st, cap ? cudaEventRecordExternal : 0));
  c->st_used[slot] = true;
  c->staged[slot] = false;
  if (!shift) c->cache_valid = false;
  return CSC_OK;
}

csc_status csc_iterate_staged(csc_ctx* c, int slot, float* x, float* d, float* z, float lambda, float step_z,
                              float step_d, double p, uint64_t seed, uint32_t iter, double obj_out[3],
                              float taus_out[2]) {
  if (!c || slot < 0 || slot > 1 || !c->staged[slot]) return fail(c, CSC_ERR_ARG, "slot not staged");
  return iterate_impl(c, nullptr, slot, x, d, z, lambda, step_z, step_d, p, seed, iter, obj_out, taus_out);
}

csc_status csc_iterate(csc_ctx* c, const float* x_host, float* x, float* d, float* z, float lambda, float step_z,
                       float step_d, double p, uint64_t seed, uint32_t iter, double obj_out[3], float taus_out[2]) {
  return iterate_impl(c, x_host, -1, x, d, z, lambda, step_z, step_d, p, seed, iter, obj_out, taus_out);
}

static csc_status iterate_impl(csc_ctx* c, const float* x_host, int slot, float* x, float* d, float* z, float lambda,
                               float step_z, float step_d, double p, uint64_t seed, uint32_t iter, double obj_out[3],
                               float taus_out[2]) {
  NvtxScope nvtx_scope(c, slot >= 0 ? "csc_iterate_staged" : "csc_iterate");
  csc_status s = check_ptrs(c, x, d, z);
  if (s != CSC_OK) return s;
  if (!obj_out && slot < 0) return fail(c, CSC_ERR_ARG, "obj_out must be a host pointer to 3 doubles");
  if (!(lambda >= 0.f) || !std::isfinite(lambda)) return fail(c, CSC_ERR_ARG, "lambda must be finite and >= 0");
  if (!(step_z >= 0.f) || !std::isfinite(step_z) || !(step_d >= 0.f) || !std::isfinite(step_d))
    return fail(c, CSC_ERR_ARG, "steps must be finite and >= 0");
  if (!(p > 0.0 && p <= 1.0)) return fail(c, CSC_ERR_ARG, "p must be in (0, 1]");
  CSC_CUDA(c, cudaSetDevice(c->device));
  if ((x_host || slot >= 0) && c->g.N > 0) {
    // new images into x.  When the residual cache holds r = D z - x_old for these (d, z) -- the
    // previous iteration's objective pass, or z = 0 -- move it to the new images without a dense
    // pass: r <- (r + x_old) - x_new (a3', linearity)
    const bool shift = c->cache_valid && c->cx == x && c->cz == z && (c->cd == d || c->cd == nullptr);
    if (slot >= 0) {
      // staged images (csc_stage_images): the H2D copy ran on the copy stream, overlapped with the
      // previous iteration; wait for it, then one pass moves the residual and copies the images in
      CSC_CUDA(c, cudaStreamWaitEvent(c->st, c->st_ready[slot], 0));
      CSC_LAUNCH(c, 1, csc::launch_stage_swap(c->stage[slot], x, c->r, n_pix(c->g), shift, c->st));
      CSC_CUDA(c, cudaEventRecord(c->st_free[slot], c->st));
      c->st_used[slot] = true;
      c->staged[slot] = false;
    } else {
      if (shift) CSC_LAUNCH(c, 1, csc::launch_resid_shift(x, c->r, n_pix(c->g), 1.f, c->st));
      CSC_CUDA(c, cudaMemcpyAsync(x, x_host, sizeof(float) * n_pix(c->g), cudaMemcpyHostToDevice, c->st));
      if (shift) CSC_LAUNCH(c, 1, csc::launch_resid_shift(x, c->r, n_pix(c->g), -1.f, c->st));
    }
    if (!shift) c->cache_valid = false;
  }
  s = csc_code_step(c, x, d, z, lambda, step_z, p, seed, iter, nullptr);
  if (s != CSC_OK) return s;
  s = csc_filter_step(c, x, d, z, step_d, nullptr);
  if (s != CSC_OK) return s;
  if (!obj_out) {  // pipelined call (csc_iterate_staged_async): the objective pass only, no host read
    s = dense_residual(c, x, d, z, true);
    if (s != CSC_OK) return s;
    return allreduce_d(c, c->dscal + kSqR, 2);
  }
  s = objective_enqueue(c, x, d, z);
  if (s != CSC_OK) return s;
  s = objective_finish(c, lambda, obj_out);
  if (taus_out) {
    taus_out[0] = c->h_fscal[kTauZ];
    taus_out[1] = c->h_fscal[kTauD];
  }
  return s;
}

// results of the pipelined slot k (its event has completed)
static csc_status res_read(csc_ctx* c, int k, double obj[3], float taus[2]) {
  CSC_CUDA(c, cudaEventSynchronize(c->res_ev[k]));
  const double half = 0.5 * c->h_res_d[k][kSqR];
  const double l1 = static_cast<double>(c->res_lam[k]) * c->h_res_d[k][kL1];
  if (obj) {
    obj[0] = half + l1;
    obj[1] = half;
    obj[2] = l1;
  }
  if (taus) {
    taus[0] = c->h_res_f[k][kTauZ];
    taus[1] = c->h_res_f[k][kTauD];
  }
  if (!std::isfinite(half + l1)) return fail(c, CSC_ERR_NONFINITE, "objective is not finite");
  return CSC_OK;
}

csc_status csc_iterate_staged_async(csc_ctx* c, int slot, float* x, float* d, float* z, float lambda, float step_z,
                                    float step_d, double p, uint64_t seed, uint32_t iter, double obj_prev[3],
                                    float taus_prev[2], int* have_prev) {
  if (!c || slot < 0 || slot > 1 || !c->staged[slot]) return fail(c, CSC_ERR_ARG, "slot not staged");
  if (!have_prev) return fail(c, CSC_ERR_ARG, "have_prev must be a host pointer");
  *have_prev = 0;
  CSC_CUDA(c, cudaSetDevice(c->device));
  if (c->h_res_d[0] == nullptr) {
    for (int i = 0; i < 2; ++i) {
      CSC_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_res_d[i]), kScalBytes));
      c->h_res_f[i] = reinterpret_cast<float*>(c->h_res_d[i] + kNumD);
      CSC_CUDA(c, cudaEventCreateWithFlags(&c->res_ev[i], cudaEventDisableTiming));
    }
  }
  const int k = c->res_next;
  if (c->res_pending == k) return fail(c, CSC_ERR_ARG, "internal: result slot still pending");
  double dummy[3];
  (void)dummy;
  csc_status s = iterate_impl(c, nullptr, slot, x, d, z, lambda, step_z, step_d, p, seed, iter, nullptr, nullptr);
  if (s != CSC_OK) return s;
  CSC_CUDA(c, cudaMemcpyAsync(c->h_res_d[k], c->dscal, kScalBytes, cudaMemcpyDeviceToHost, c->st));
  CSC_CUDA(c, cudaEventRecord(c->res_ev[k], c->st));
  c->res_lam[k] = lambda;
  const int prev = c->res_pending;
  c->res_pending = k;
  c->res_next = k ^ 1;
  if (prev >= 0) {
    s = res_read(c, prev, obj_prev, taus_prev);
    if (s != CSC_OK) return s;
    *have_prev = 1;
  }
  return CSC_OK;
}

csc_status csc_iterate_drain(csc_ctx* c, double obj[3], float taus[2], int* have) {
  if (!c || !have) return fail(c, CSC_ERR_ARG, "have must be a host pointer");
  *have = 0;
  if (c->res_pending < 0) return CSC_OK;
  const int k = c->res_pending;
  c->res_pending = -1;
  csc_status s = res_read(c, k, obj, taus);
  if (s != CSC_OK) return s;
  *have = 1;
  return CSC_OK;
}

csc_status csc_mask_bits(csc_ctx* c, uint32_t iter, double p, uint64_t seed, uint32_t* bits_dev) {
  if (!c || !aligned4(bits_dev)) return fail(c, CSC_ERR_ARG, "bits_dev must be a device pointer");
  if (!(p > 0.0 && p <= 1.0)) return fail(c, CSC_ERR_ARG, "p must be in (0, 1]");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const uint64_t thr = static_cast<uint64_t>(std::floor(p * 4294967296.0));
  CSC_LAUNCH_C(c, CSC_K_MASK, 1, csc::launch_mask_bits(c->g, seed, iter, thr, bits_dev, c->st, c->mask_mode));
  return CSC_OK;
}

csc_status csc_mask_selwords(csc_ctx* c, uint32_t iter, double p, uint64_t seed, uint32_t* words_dev,
                             int32_t info[4]) {
  if (!c || !info) return fail(c, CSC_ERR_ARG, "info (host, 4 ints) required");
  if (!(p > 0.0 && p <= 1.0)) return fail(c, CSC_ERR_ARG, "p must be in (0, 1]");
  if (!c->ct_on) return fail(c, CSC_ERR_SHAPE, "the code step of this context does not use selection words");
  info[0] = c->ct.nkg;
  info[1] = c->ct.wper;
  info[2] = c->ct.wnc;
  info[3] = c->ct.KC;
  if (words_dev == nullptr) return CSC_OK;
  if (!aligned4(words_dev)) return fail(c, CSC_ERR_ARG, "words_dev must be a device pointer");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const uint64_t thr = static_cast<uint64_t>(std::floor(p * 4294967296.0));
  CSC_LAUNCH_C(c, CSC_K_MASK, 1, csc::launch_mask_selwords(c->g, c->ct, seed, iter, thr, words_dev, c->st, c->mask_mode));
  return CSC_OK;
}

csc_status csc_read_scalars(csc_ctx* c, double out[4]) {
  if (!c || !out) return fail(c, CSC_ERR_ARG, "out (host, 4 doubles) required");
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_CUDA(c, cudaMemcpyAsync(c->h_dscal, c->dscal, sizeof(double) * kNumD, cudaMemcpyDeviceToHost, c->st));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  out[0] = c->h_dscal[kSqR];
  out[1] = c->h_dscal[kL1];
  out[2] = c->h_dscal[kZg2];
  out[3] = c->h_dscal[kGG];
  return CSC_OK;
}

csc_status csc_zg_sumsq(csc_ctx* c, const float* z, const double* g_dev) {
  if (!c || !g_dev || (c->g.N > 0 && !aligned4(z))) return fail(c, CSC_ERR_ARG, "z and g_dev must be device pointers");
  CSC_CUDA(c, cudaSetDevice(c->device));
  const Geom& g = c->g;
  CSC_CUDA(c, cudaMemcpyAsync(c->gsum, g_dev, sizeof(double) * g.K * g.S * g.S, cudaMemcpyDeviceToDevice, c->st));
  CSC_LAUNCH(c, 1, csc::launch_grad_finish(g, c->gsum, c->g32, c->dscal + kGG, c->gf_scratch, c->st));
  return zg_pass(c, z);
}

csc_status csc_read_residual(csc_ctx* c, float* r_dev) {
  if (!c || (c->g.N > 0 && !aligned4(r_dev))) return fail(c, CSC_ERR_ARG, "r_dev must be a device pointer");
  CSC_CUDA(c, cudaSetDevice(c->device));
  if (c->g.N > 0)
    CSC_CUDA(c, cudaMemcpyAsync(r_dev, c->r, sizeof(float) * n_pix(c->g), cudaMemcpyDeviceToDevice, c->st));
  return CSC_OK;
}

csc_status csc_read_grad(csc_ctx* c, double* g_dev) {
  if (!c || !g_dev) return fail(c, CSC_ERR_ARG, "g_dev must be a device pointer");
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_CUDA(c, cudaMemcpyAsync(g_dev, c->gsum, sizeof(double) * c->g.K * c->g.S * c->g.S, cudaMemcpyDeviceToDevice,
                              c->st));
  return CSC_OK;
}

csc_status csc_count_nonzero(csc_ctx* c, const float* v, int64_t n, uint64_t* count) {
  if (!c || !count || n < 0 || (n > 0 && !aligned4(v))) return fail(c, CSC_ERR_ARG, "v (device), n >= 0, count (host)");
  CSC_CUDA(c, cudaSetDevice(c->device));
  if (!c->cnt_dev) CSC_CUDA(c, cudaMalloc(&c->cnt_dev, sizeof(uint64_t)));
  CSC_CUDA(c, cudaMemsetAsync(c->cnt_dev, 0, sizeof(uint64_t), c->st));
  if (n > 0) CSC_LAUNCH(c, 1, csc::launch_count_nonzero(v, n, c->cnt_dev, c->st));
  CSC_CUDA(c, cudaMemcpyAsync(c->h_dscal + kCnt, c->cnt_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  std::memcpy(count, c->h_dscal + kCnt, sizeof(uint64_t));
  return CSC_OK;
}

csc_status csc_set_nvtx(csc_ctx* c, int enable) {
  if (!c) return CSC_ERR_ARG;
  c->nvtx = enable != 0;
  return CSC_OK;
}

csc_status csc_comm_check(csc_ctx* c) {
  if (!c) return CSC_ERR_ARG;
  if (c->world <= 1 || c->comm == nullptr) return CSC_OK;
  if (!g_nccl.CommGetAsyncError) return fail(c, CSC_ERR_NCCL, "libnccl.so.2 lacks ncclCommGetAsyncError");
  ncclResult_t ar = ncclSuccess;
  const ncclResult_t r = g_nccl.CommGetAsyncError(c->comm, &ar);
  if (r != ncclSuccess) return fail(c, CSC_ERR_NCCL, std::string("ncclCommGetAsyncError: ") + g_nccl.GetErrorString(r));
  if (ar != ncclSuccess && ar != ncclInProgress)
    return fail(c, CSC_ERR_NCCL, std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(ar));
  return CSC_OK;
}

csc_status csc_lipschitz(csc_ctx* c, const float* d, double* out) {
  if (!c || !aligned4(d) || !out) return fail(c, CSC_ERR_ARG, "d (device) and out (host) required");
  CSC_CUDA(c, cudaSetDevice(c->device));
  CSC_LAUNCH_C(c, CSC_K_LIPSCHITZ, 2, csc::launch_lipschitz(c->g, d, c->lip_part, c->dscal + kLhat, nullptr, c->st));
  c->lip_valid = false;  // kLhat now describes this d
  CSC_CUDA(c, cudaMemcpyAsync(c->h_dscal + kLhat, c->dscal + kLhat, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CSC_CUDA(c, cudaStreamSynchronize(c->st));
  *out = c->h_dscal[kLhat];
  return CSC_OK;
}

}  // extern "C"

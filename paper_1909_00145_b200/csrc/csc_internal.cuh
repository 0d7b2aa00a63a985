// csc_internal.cuh -- internal launch interface between the C ABI (csc_api.cu)
// and the sm_100a kernels (csc_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

namespace csc {

// A 2D TMA tensor map cached with the pointer / shape it encodes.  Owned by a context (csc_ctx), so
// contexts on different devices or threads never share one (include/csc.h: one context per
// (rank, device, stream)).
struct TmapCache {
  const void* ptr = nullptr;
  uint64_t key[4] = {0, 0, 0, 0};
  bool valid = false;
  alignas(64) CUtensorMap map;
};
// Encode (or reuse) a 2D tiled map: dims {d0 (contiguous), d1}, row stride stride1 bytes, box {b0, b1};
// no interleave, zero fill out of bounds.  cudaErrorNotSupported when the driver entry point is absent,
// cudaErrorInvalidValue when the shape / alignment is not encodable.
cudaError_t tmap_2d(TmapCache& c, CUtensorMapDataType dt, const void* ptr, uint64_t d0, uint64_t d1, uint64_t stride1,
                    uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw, CUtensorMapL2promotion promo);
bool tmap_available();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (function, device): the attribute is a
// per-device setting, so a process-wide flag would leave a second device unconfigured.
cudaError_t set_smem_attr_once(const void* func, int bytes);

struct Geom {
  int N, K, S, H, W, Hc, Wc, P;
};

// ---- tiling constants shared by launcher and kernels ----
constexpr int kConvTX = 8, kConvTY = 16, kConvR = 4, kConvC = 8;
constexpr int kConvTW = kConvTX * kConvC;  // 64 output columns per tile
constexpr int kConvTH = kConvTY * kConvR;  // 64 output rows per tile
constexpr int kConvThreads = kConvTX * kConvTY;

constexpr int kWgTX = 8, kWgTY = 16, kWgRB = 4, kWgC = 8;
constexpr int kWgTW = kWgTX * kWgC;  // 64
constexpr int kWgTH = kWgTY * kWgRB; // 64
constexpr int kWgThreads = kWgTX * kWgTY;

constexpr int kCodeWarps = 4;
constexpr int kCodeThreads = 32 * kCodeWarps;
constexpr int kCodePitch = 64;  // r-tile pitch in floats; multiple of 32 => lane L hits bank L+b

constexpr int kReduceThreads = 256;
constexpr int kFinalizeBlocks = 148 * 4;

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Filter sizes with compiled kernels.
inline bool filter_size_supported(int s) {
  return s == 1 || s == 3 || s == 5 || s == 7 || s == 9 || s == 11;
}

// All launchers return cudaGetLastError() of their launch.
// Code-step launchers: tau_stride 0 -> tau_dev[0] for every filter; 1 -> tau_dev[k] (ESO rule).
// kConvResidual: out = y - x (plain y when x == nullptr); kConvSumSq: only sum y^2.
enum ConvMode : int { kConvResidual = 0, kConvSumSq = 1 };

// y = sum_{k in [k0,k1)} f_k * z_k (valid true convolution) for all images.
// ksplit == 1: out = y - x (mode residual, stored to r) or nothing (sumsq);
//   per-block fp64 partials of sum(out^2) -> sq_part[blocks], of |z| over owned
//   code positions -> l1_part[blocks] (if l1_part != nullptr).
// ksplit > 1: y of split ks -> part[ks][N][H][W]; finalize with launch_conv_finalize.
cudaError_t launch_conv_fwd(const Geom& g, const float* z, const float* filt, const float* x,
                            float* r, float* part, int ksplit, int mode, double* sq_part,
                            double* l1_part, cudaStream_t st, int* nblocks_out);
int conv_fwd_blocks(const Geom& g, int ksplit);
cudaError_t launch_conv_finalize(const Geom& g, const float* part, int ksplit, const float* x,
                                 float* r, int mode, double* sq_part, cudaStream_t st);

// Fixed-order fp64 sum of n partials -> *out (single block).  scale applied to result.
cudaError_t launch_reduce_sum(const double* part, int n, double* out, double scale,
                              cudaStream_t st);

// Filter-gradient partials: gpart[G][K][S*S] (fp64); grid (G, K).
cudaError_t launch_wgrad(const Geom& g, const float* z, const float* r, int G, double* gpart,
                         cudaStream_t st);
// gsum[K*S*S] = sum_G gpart (fixed order, fp64).
cudaError_t launch_wgrad_reduce(const Geom& g, const double* gpart, int G, double* gsum,
                                cudaStream_t st);
// g32 = (float)gsum, gg_out = sum gsum^2 (fp64) -- after the cross-rank all-reduce.
// scratch: ceil(K s^2 / 256) + 1 doubles, the last one zero (a block counter the kernel clears)
cudaError_t launch_grad_finish(const Geom& g, const double* gsum, float* g32, double* gg_out, double* scratch,
                               cudaStream_t st);

// Mask (Philox4x32-10) -- internal column-word layout for the code step:
//   colw[(k*NB + ub)*Wc + v] bit r = mask(k, 32*ub + r, v), NB = ceil(Hc/32).
// mode 0: per-entry Bernoulli (Eq.2); mode 1: one draw per aligned 8-coordinate block (E5)
// iter_off (device, nullable): the mask iteration is iter + *iter_off, read at launch (graph replays)
cudaError_t launch_mask_colwords(const Geom& g, uint64_t seed, uint32_t iter, uint64_t thr,
                                 uint32_t* colw, cudaStream_t st, int mode = 0, const uint32_t* iter_off = nullptr);
// Canonical layout for the test hook.
cudaError_t launch_mask_bits(const Geom& g, uint64_t seed, uint32_t iter, uint64_t thr,
                             uint32_t* bits, cudaStream_t st, int mode = 0);

// Masked proximal-gradient code step.
// zmax (may be null): raised (atomicMax of float bits) to >= |z| of every code written.
// ESO step rule: tauk[k] = fp32(1 / (p * lhat + (1-p) ||d_k||^2))
cudaError_t launch_eso_tau(const Geom& g, const float* d, double p, const double* lhat, float* tauk, cudaStream_t st);
cudaError_t launch_code_step(const Geom& g, const float* r, const float* d, float* z,
                             const uint32_t* colw, int all_selected, const float* tau_dev,
                             float lam, uint32_t* zmax, cudaStream_t st,
                             int tau_stride = 0);

// L_D(d) = max over 64x64 DFT grid of sum_k |d^_k|^2 -> lhat (fp64), and
// tau_out = (float)(1/L) if tau_out != nullptr.  part: >= 64 doubles scratch.
cudaError_t launch_lipschitz(const Geom& g, const float* d, double* part, double* lhat,
                             float* tau_out, cudaStream_t st);

// tau_d = step > 0 ? step : (zg2 > 0 ? (float)(gg/zg2) : 0)  (device scalar).
cudaError_t launch_filter_tau(const double* gg, const double* zg2, float step, float* tau_d,
                              cudaStream_t st);
// d_k <- (float)((d_k - tau g_k) / max(1, ||d_k - tau g_k||)) in fp64.
cudaError_t launch_filter_update(const Geom& g, float* d, const double* gsum, const float* tau_d,
                                 cudaStream_t st);

// *p = v on the stream (a kernel argument, not a pageable host copy: capturable in a CUDA graph).
cudaError_t launch_set_f32(float* p, float v, cudaStream_t st);
// dst[0..n) = *src
cudaError_t launch_bcast_f32(float* dst, const float* src, int n, cudaStream_t st);

// r = -x (zero codes).
cudaError_t launch_neg_copy(const float* x, float* r, int64_t n, cudaStream_t st);
// r += sign * x
cudaError_t launch_count_nonzero(const float* v, int64_t n, uint64_t* out, cudaStream_t st);
cudaError_t launch_resid_shift(const float* x, float* r, int64_t n, float sign, cudaStream_t st);
// x <- xn and, when shift, r <- (r + x_old) - xn in one pass (csc_iterate_staged)
cudaError_t launch_stage_swap(const float* xn, float* x, float* r, int64_t n, bool shift, cudaStream_t st);

// ---- tensor-core (tcgen05, 3xTF32) dense pass, csc_tc.cu
constexpr int kTcMaxKC = 104;  // filters per k-split held resident in shared memory
struct TcPlan {
  int NT, natoms, nks, KC, NCH, SEGR, RW, BR, nbands, nitems, grid, smem;
  size_t part_floats, bimg_floats;
  int WL;    // SS kernels: band window length (floats)
  bool ss;   // true: the TMA-fed SS kernel (csc_conv_ss.cu) runs this plan
  bool half; // true: the fp16-split SS kernel (csc_conv_h.cu) runs this plan
  const int* sched = nullptr;  // half: device copy of conv_h_schedule (owned by the context), or round robin
};
int tc_ntaps_padded(int S);
// filter taps -> B image bimg[nks][hi|lo][natoms][KC][32] (MN-major SWIZZLE_128B_BASE32B)
cudaError_t launch_tc_bimg(const Geom& g, const TcPlan& p, const float* filt, float* bimg, cudaStream_t st);
// TMA-fed SS dense pass (csc_conv_ss.cu): Hc*Wc % 4 == 0, s in {5,7,9,11}
bool conv_ss_supported(const Geom& g);
bool conv_ss_plan(const Geom& g, int num_sms, TcPlan& p);
cudaError_t launch_conv_ss(const Geom& g, const TcPlan& p, TmapCache* tmc, const float* z, const float* bimg,
                           float* part, double* l1_part, cudaStream_t st);
// fp16-split SS dense pass (csc_conv_h.cu): Wc >= 128, Hc*Wc % 4 == 0.  zmax: upper bound of max|z|
// (float bits, device); fmax: written with max|filt| (float bits, device).
bool conv_h_supported(const Geom& g);
bool conv_h_plan(const Geom& g, int num_sms, TcPlan& p);
// LPT assignment of the (image, band of BR code rows) items to G CTAs, cost = 128-position tiles + overhead:
// returns the busiest CTA's cost; out (if any) = [G + 1] CTA offsets, then the items CTA by CTA
int64_t lpt_bands(const Geom& g, int BR, int G, int overhead, std::vector<int>* out);
// the balanced item schedule of a conv_h plan: [grid + 1] CTA offsets, then the items CTA by CTA
void conv_h_schedule(const Geom& g, const TcPlan& p, std::vector<int>& out);
// build_b = false reuses the fp16 filter image (and fmax) of the previous call with the same filt.
// precise: hi*hi and the cross products accumulate in separate TMEM accumulators (the ||Zg||^2 pass,
// DESIGN.md reading T3).  tmc: the context's cached tensor map of z.
cudaError_t launch_conv_h(const Geom& g, const TcPlan& p, TmapCache* tmc, const float* z, const float* filt,
                          float* bimg, const uint32_t* zmax, uint32_t* fmax, float* part, double* l1_part,
                          cudaStream_t st, bool build_b = true, bool precise = false);
// *out = bits of max |x[i]| (atomicMax over non-negative float bits; resets *out first)
cudaError_t launch_absmax(const float* x, int64_t n, uint32_t* out, cudaStream_t st);
bool conv_tc_supported(const Geom& g);
TcPlan conv_tc_plan(const Geom& g, int num_sms);
// y (all k-splits) -> band partial windows in part; per-CTA |z| partials -> l1_part[nks*grid] if non-null.
cudaError_t launch_conv_tc(const Geom& g, const TcPlan& p, const float* z, const float* filt, float* bimg,
                           float* part, double* l1_part, cudaStream_t st);
// part -> r = y - x (residual mode) or sum y^2 (sum-of-squares mode); per-block partials -> sq_part[kFinalizeBlocks].
// the fixup's own reductions (fsum != nullptr): sum r^2 -> out_sq and sum of the nl1 partials l1_part
// -> out_l1 (optional), in fixed orders; counter: one zero-initialised 64-bit word the launch clears
struct FixupSums {
  double* out_sq = nullptr;
  const double* l1_part = nullptr;
  int nl1 = 0;
  double* out_l1 = nullptr;
  unsigned long long* counter = nullptr;
};
cudaError_t launch_conv_tc_fixup(const Geom& g, const TcPlan& p, const float* part, const float* x, float* r,
                                 int mode, double* sq_part, cudaStream_t st, const FixupSums* fsum = nullptr);


// ---- tensor-core (tcgen05, 3xTF32) filter gradient, csc_wgrad_tc.cu
struct WgTcPlan {
  int KC, Npad, nkg, G, L, nseg, nitems, pitch, rs_rows, rs_floats, stage_bytes;
  int grid, smem;
};
bool wgrad_tc_supported(const Geom& g);
WgTcPlan wgrad_tc_plan(const Geom& g, int num_sms);
// Per-CTA fp64 partials gpart[p.G][K][S*S] (reduce with launch_wgrad_reduce(g, gpart, p.G, ...)).
// z must be 16-byte aligned.
cudaError_t launch_wgrad_tc(const Geom& g, const WgTcPlan& p, TmapCache* tmc, const float* z, const float* r,
                            double* gpart, cudaStream_t st);


// ---- tensor-core filter gradient at the fp16 rate (kind::f16, 3-term split), csc_wgrad_h.cu
struct WhPlan {
  int KC, Npad, NCH, nkg, G, L, nseg, nitems, pitch, rs_rows, rs_floats, NB, NR, cpt;
  int grid, smem;
  bool ok;
};
bool wgrad_h_supported(const Geom& g);
WhPlan wgrad_h_plan(const Geom& g, int num_sms);
// Per-CTA fp64 partials gpart[p.G][K][S*S] as launch_wgrad_tc; zmax bounds max|z|, rmax = max|r| (float bits).
cudaError_t launch_wgrad_h(const Geom& g, const WhPlan& p, TmapCache* tmc, const float* z, const float* r,
                           const uint32_t* zmax, const uint32_t* rmax, double* gpart, cudaStream_t st);

// ---- tensor-core (tcgen05, 3xTF32) dense-then-mask code step, csc_code_tc.cu
struct CodeTcPlan {
  int KC, Npad, nkg, G, L, nseg, nitems, pitch, rs_rows, rs_floats, b_bytes;
  size_t sw_words;  // selection-word mask size (wper * nkg * Hc * Wc words)
  int wnc, wper;    // selection words: wnc filters per word, wper word blocks per filter group
  int grid, smem;
  bool ok;
  bool half;        // true: the fp16-split kernel (csc_code_h.cu)
  // csc_code_h.cu: items are bands of BR code rows; ngroups 16-filter groups per filter group;
  // a3' band partials [nkg][N][nbands][BR+P][W] (a3_floats)
  int ngroups, BR, nbands, WL;
  size_t a3_floats;
  const int* sched = nullptr;  // device copy of code_h_schedule (owned by the context), or round robin
};
bool code_tc_supported(const Geom& g);
CodeTcPlan code_tc_plan(const Geom& g, int num_sms);
// Mask as selection words sw[wper*nkg][Hc*Wc]: bit i of sw[kg*wper+cb][p] = mask(kg*KC + cb*wnc + i, p).
cudaError_t launch_mask_selwords(const Geom& g, const CodeTcPlan& p, uint64_t seed, uint32_t iter, uint64_t thr,
                                 uint32_t* words, cudaStream_t st, int mode = 0, const uint32_t* iter_off = nullptr);
// fp16-split variant (csc_code_h.cu): Hc*Wc % 4 == 0 (TMA view of z); rmax = max|r| (float bits).
bool code_h_supported(const Geom& g);
CodeTcPlan code_h_plan(const Geom& g, int num_sms);
// the balanced item schedule of a code_h plan (the G CTAs of one filter group; every group runs the same list)
void code_h_schedule(const Geom& g, const CodeTcPlan& p, std::vector<int>& out);
// a3_part != nullptr (and !plain): the incremental residual r' = r + D dz is written as band partials
// [nkg][N][nbands][BR+P][W]; launch_code_a3_fixup then adds them to r (a3').
cudaError_t launch_code_h(const Geom& g, const CodeTcPlan& p, TmapCache* tmc, const float* r, const float* d,
                          float* z, const uint32_t* words, const float* tau_dev, float lam, const uint32_t* rmax,
                          uint32_t* zmax, cudaStream_t st,
                          bool plain = false, int tau_stride = 0, float* a3_part = nullptr);
cudaError_t launch_code_a3_fixup(const Geom& g, const CodeTcPlan& p, const float* part, float* r, cudaStream_t st);
// words == nullptr: every code selected (p = 1).
cudaError_t launch_code_tc(const Geom& g, const CodeTcPlan& p, const float* r, const float* d, float* z,
                           const uint32_t* words, const float* tau_dev, float lam, uint32_t* zmax, cudaStream_t st,
                             int tau_stride = 0);

// ADMM masked-LASSO code solver (csc_admm.cu).  Vectors are compact [N][ms] (ms = mc rounded up
// to 4, pads 0) over the selected positions idx[0..mc) of the (image-shared) mask; per-block
// partials `part` hold N * max(admm_blocks(g, ms), admm_dtr_blocks(g)) doubles; per-image scalars
// are N doubles.
int admm_blocks(const Geom& g, int64_t ms);
int admm_dtr_blocks(const Geom& g);
int admm_idx_blocks(const Geom& g);
// bits (canonical layout) -> idx (ascending positions), woff[w] = set bits before word w,
// *mc (device) = popcount; cnt/off: admm_idx_blocks entries
cudaError_t launch_admm_index(const Geom& g, const uint32_t* bits, uint32_t* cnt, uint64_t* off, uint64_t* mc,
                              uint32_t* idx, uint32_t* woff, cudaStream_t st);
// row_off[r] (r in [0, K*Hc]) = first compact index of code row r = k*Hc + u
cudaError_t launch_admm_row_off(const Geom& g, const uint32_t* idx, int64_t mc, uint64_t* row_off,
                                cudaStream_t st);
// SIMT masked correlation: out = sign * M D^T e (+ rho v, and part[N][admm_dtr_blocks] = per-block
// sum v*out, when v != null)
cudaError_t launch_masked_dtr(const Geom& g, const uint32_t* idx, const uint64_t* row_off, int64_t ms, const float* e,
                              const float* d, const float* v, float rho, float sign, float* out, double* part,
                              cudaStream_t st);
// out = sign * Cd[idx] (+ rho v, part[N][admm_blocks] = per-block sum v*out, when v != null)
cudaError_t launch_admm_gather(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* Cd,
                               const float* v, float rho, float sign, float* out, double* part, cudaStream_t st);
cudaError_t launch_admm_init(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* z, float* W,
                             float* Y, cudaStream_t st);
// Zd (dense, zeros off the mask) <- R, or with PV != null the CG direction PV = R + beta PV
// (beta = rr_new/rr per image; PV = R when rr == null).  max|written| -> atomicMax(bound).
cudaError_t launch_admm_expand(const Geom& g, const uint32_t* bits, const uint32_t* woff, int64_t ms, const float* R,
                               float* PV, const double* rr, const double* rr_new, float* Zd, uint32_t* bound,
                               cudaStream_t st);
// z[idx] = Y (selected positions only); max|written| -> atomicMax(bound) when bound != null
cudaError_t launch_admm_scatter(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* Y, float* z,
                                uint32_t* bound, cudaStream_t st);
// rr[n] = |R_n|^2 (fixed-order fp64)
cudaError_t launch_sumsq(const Geom& g, int64_t ms, const float* R, double* part, double* rr, cudaStream_t st);
// Explicit CG residual R = ATB + rho (Y - U) - Q (init: ATB = R + Q - rho Y); rr[n] = |R_n|^2
cudaError_t launch_cg_resid(const Geom& g, int64_t ms, float* ATB, const float* Y, const float* U, const float* Q,
                            float rho, float* R, double* part, double* rr, bool init, cudaStream_t st);
// part_pq: nb_pq partials per image (admm_dtr_blocks for masked_dtr, admm_blocks for gather)
cudaError_t launch_cg_step(const Geom& g, int64_t ms, const double* rr, const double* part_pq, int nb_pq, float* W,
                           float* R,
                           const float* PV, const float* Q, double* part_rr, double* rr_new, cudaStream_t st);
// ADMM update (over-relaxed, shrinkage, dual) carrying the CG residual R to the new right-hand
// side; rr[n] = |R_n|^2 afterwards
cudaError_t launch_admm_update(const Geom& g, int64_t ms, const float* W, float* Y, float* U, float* R, float alpha,
                               float kappa, float rho, double* part, double* rr, cudaStream_t st);

// Projected block-coordinate filter update (csc_bcd.cu).  gpart: K * bcd_gram_splits * M * M
// doubles (the per-rank Gram partials; all-reduce them for world > 1), ainv: K * M * M doubles,
// flags: K bytes (1 = filter left unchanged), part: bcd_gk_blocks * M doubles, gk / dl: M doubles.
int bcd_gram_splits(const Geom& g);
int bcd_gk_blocks(const Geom& g);
cudaError_t launch_bcd_gram(const Geom& g, const float* z, double* gpart, cudaStream_t st);
cudaError_t launch_bcd_inverse(const Geom& g, const double* gpart, double ridge_rel, double* ainv, uint8_t* flags,
                               cudaStream_t st);
cudaError_t launch_bcd_gk(const Geom& g, int k, const float* z, const float* r, double* part, double* gk,
                          cudaStream_t st);
cudaError_t launch_bcd_update(const Geom& g, int k, const double* gk, const double* ainv, const uint8_t* flags,
                              float* d, double* dl, const float* z, float* r, cudaStream_t st);

// Lag-structured Gram blocks (csc_bcd.cu; needs H, W > P): gq = bcd_lag_bytes scratch, cfull =
// K*M*M doubles (the full C_kk), then launch_bcd_inverse_full.
bool bcd_lag_supported(const Geom& g);
size_t bcd_lag_bytes(const Geom& g);
cudaError_t launch_bcd_lag_gram(const Geom& g, const float* z, double* gq, double* cfull, cudaStream_t st);
cudaError_t launch_bcd_inverse_full(const Geom& g, const double* cfull, double ridge_rel, double* ainv,
                                    uint8_t* flags, cudaStream_t st);
// Online surrogates (csc_bcd.cu): C block-major [K][K][M][M], B [K][M] (fp64).  pp: K(K+1)/2 *
// sur_gram_splits * M * M doubles; C <- wo C + wn (batch Gram), B <- wo B + wn (batch Z^T x).
// pp == nullptr selects the lag-structured pair kernel (needs bcd_lag_supported), folded in place.
int sur_gram_splits(const Geom& g);
cudaError_t launch_sur_update(const Geom& g, const float* x, const float* z, double* pp, double* part, double* gk,
                              double wo, double wn, double* C, double* B, cudaStream_t st);
// diag (K M M doubles) <- the diagonal blocks; ainv / flags as launch_bcd_inverse
cudaError_t launch_sur_prepare(const Geom& g, const double* C, double* diag, double ridge_rel, double* ainv,
                               uint8_t* flags, cudaStream_t st);
// one Eq.8 block step for filter k (gk, dl: M doubles)
cudaError_t launch_sur_filter(const Geom& g, int k, const double* C, const double* B, const double* ainv,
                              const uint8_t* flags, float* d, double* gk, double* dl, cudaStream_t st);

}  // namespace csc

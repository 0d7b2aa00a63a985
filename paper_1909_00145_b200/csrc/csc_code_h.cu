// csc_code_h.cu -- masked proximal-gradient code step, dense-then-mask on the sm_100a tensor cores
// with the 3-term fp16 split (tcgen05.mma kind::f16), fused with the incremental residual (a3').
//
// Code step (Eq.3-4, §3.1, shrinkage P:311-312, R1/R2):
//   for every masked code (k, u, v) of image n:  c = sum_{a,b} d[k,a,b] r[n,u-P+a,v-P+b],
//   z <- S_{tau lambda}(z - tau c);  unmasked codes are untouched.
// Incremental residual (SURVEY.md §8(a) a3'; linearity of D):
//   r' = r + sum_k d_k * (z_new - z_old)_k,  so the filter step needs no dense residual pass.
//
// Per 128-position tile of a band of BR code rows (flattened positions p = u*Wc + v):
//   GEMM 1 (the correlation):  C[p][k] = sum_t R[p][t] d[k][t], M = 128 positions, N = Npad filters,
//     K = 128 taps (8 K16-steps).  A = im2col(r) in TMEM (lane = position, two fp16 taps per column),
//     written by the converter warps from the band's residual rows (cp.async staging); B = the filters,
//     K-major SWIZZLE_128B fp16, resident.
//   epilogue (16 warps = 4 TMEM lane quarters x 4): warp (q, j) owns the 16-filter groups (j + t) mod 4
//     and +4 of tile t (rotated so the 7 groups of Npad = 112 spread evenly).  Only the codes the mask
//     selects are read: each lane cp.async's the 4-byte codes whose selection bit is set, one tile
//     ahead, so HBM moves the 32-B sectors that hold a selected code and nothing else (the cost falls
//     with p).  It applies step / shrinkage, stores the codes that change, and writes
//     dz = z_new - z_old (0 elsewhere) as fp16 hi/lo into the accumulator columns it has just read:
//     K16-step g of the second GEMM takes hi from columns 16g..16g+7 and lo from 16g+8..16g+15, exactly
//     the columns of C for filters 16g..16g+15, so no warp overwrites a column another warp still reads.
//   GEMM 2 (the increment):  Y[p][t] = sum_k dz[p][k] d[k][t], M = 128, N = 128 taps, K = Npad filters;
//     A = dz in TMEM, B = the same resident filter image read MN-major (taps contiguous).
//   col2im (4 warps, one per lane quarter): as the dense pass (csc_conv_h.cu), one rotation shuffle per
//     tap into the band window; the window is flushed per band to partials [kg][n][band][BR+P][W] that
//     launch_code_a3_fixup adds to r in a fixed order.
// Operands are split after exact power-of-two scalings (reading T6): x_s = x 2^e,
// hi = rn11(x_s) (an exact fp16), lo = fp16_rn(x_s - hi); products hi*hi + hi*lo + lo*hi accumulate
// in fp32.  e_r from max|r|, e_d from max|d| of the CTA's filter group, e_dz from the bound
// |dz| <= tau (||d_k||_1 max|r| + lambda) (one step of the prox-gradient map, |S(w) - z| <= |w - z| +
// kappa), which keeps every scaled value <= 2^14 with 2^17 of headroom below for full precision.
// CTA (persistent, 25 warps): warp 0 MMA, warps 1..4 converters, 5..20 epilogue, 21..24 col2im.
// TMEM (512 columns): C / dz double buffer [0, 2 Npad), im2col slots [256, 384), Y [384, 512).
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdint>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kChNS = 2;          // im2col slots (4 K16-steps = 64 taps each) in TMEM
constexpr int kChEpiWarps = 16;  // 4 per TMEM lane quarter
constexpr int kChHelpWarps = 8;  // 2 per TMEM lane quarter: the im2col of the next tile and the col2im of the last
constexpr int kChEpiPerQ = kChEpiWarps / 4;
constexpr int kChChunks = (8 + kChEpiPerQ - 1) / kChEpiPerQ;  // 16-filter groups per warp per tile (Npad <= 128)
constexpr int kChEpiBase = 1, kChHelpBase = kChEpiBase + kChEpiWarps;
constexpr int kChWarps = kChHelpBase + kChHelpWarps;
constexpr int kChThreads = 32 * kChWarps;
constexpr int kChTile = 128;
constexpr int kChSmemMax = 226 * 1024;
constexpr uint32_t kColA = 256, kColY = 384;
constexpr int kZBuf = kChChunks * 16 * 32;  // floats per epilogue warp: chunks x 16 filters x 32 positions
constexpr int kWBuf = kChChunks * 32;       // selection words per epilogue warp

__host__ __device__ constexpr uint32_t idesc_f16_kk(int M, int N) {  // fp16 A/B K-major, fp32 D
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (0u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16_kmn(int M, int N) {  // A K-major (TMEM), B MN-major
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ int scale_exp_h(uint32_t mbits) {
  if ((mbits & 0x7FFFFFFFu) == 0u) return 0;
  const int E = static_cast<int>((mbits >> 23) & 0xFFu) - 127;
  int e = 13 - E;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}
__device__ __forceinline__ float exp2i_h(int e) { return __uint_as_float(static_cast<uint32_t>(e + 127) << 23); }
__device__ __forceinline__ float rn11_h(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ uint32_t pack_h2_h(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void cp_async4_if(uint32_t smem_dst, const float* src, bool p) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(smem_dst),
               "l"(src), "r"(p ? 1 : 0)
               : "memory");
}
// store v at base + off_bytes when sel != 0: one IMAD.WIDE for the address, the predicate from sel itself
__device__ __forceinline__ void st_off_if_nz(float* base, uint32_t off_bytes, float v, float sel) {
  asm volatile(
      "{\n.reg .pred q;\n.reg .u64 a;\nsetp.ne.f32 q, %3, 0f00000000;\nmad.wide.u32 a, %1, 1, %0;\n@q st.global.f32 [a], %2;\n}\n" ::"l"(
          base),
      "r"(off_bytes), "f"(v), "f"(sel)
      : "memory");
}
__device__ __forceinline__ void st_global_if(float* ptr, float v, bool p) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f32 [%0], %1;\n}\n" ::"l"(ptr), "f"(v),
               "r"(p ? 1 : 0)
               : "memory");
}

// Per-role cycle counters for tuning (build with -DCSC_ROLE_TIMING; off in the product build).
#ifdef CSC_ROLE_TIMING
struct RoleClock {
  unsigned long long v[7];
  unsigned long long t0;
  __device__ RoleClock() : t0(0) {
#ifdef __CUDA_ARCH__
    t0 = clock64();
#endif
    for (int i = 0; i < 7; ++i) v[i] = 0;
  }
};
#define RT_WAIT(rc, slot, stmt)                      \
  do {                                               \
    const unsigned long long _a = clock64();         \
    stmt;                                            \
    (rc).v[slot] += clock64() - _a;                  \
  } while (0)
#define RT_DUMP(rc, dbg, role)                                                          \
  do {                                                                              \
    if ((dbg) != nullptr) {                                                         \
      for (int _i = 0; _i < 7; ++_i) (dbg)[blockIdx.x * 32 + (role) * 8 + _i] = (rc).v[_i]; \
      (dbg)[blockIdx.x * 32 + (role) * 8 + 7] = clock64() - (rc).t0;               \
    }                                                                               \
  } while (0)
#else
struct RoleClock {};
#define RT_WAIT(rc, slot, stmt) stmt
#define RT_DUMP(rc, dbg, role) \
  do {                         \
  } while (0)
#endif

struct ChArgs {
  CUtensorMap tm_z;      // z as [N*K planes][Hc*Wc positions] fp32, box {32, 16}
  CUtensorMap tm_w;      // selection words [nkg*ngroups][Hc*Wc] u32, box {32, 1}
  const float* r;        // [N][H][W]
  const float* d;        // [K][S][S]
  float* z;              // [N][K][Hc][Wc]
  const uint32_t* mask;  // selection words [nkg][ngroups][plane] (bit i: filter kg*KC + 16 g + i) or nullptr (all)
  const float* tau;
  const uint32_t* rmax;  // max|r| (float bits)
  uint32_t* zmax;        // raised by every written code, or nullptr
  float* part;           // a3' band partials [nkg][N][nbands][BR+P][W], or nullptr (no a3')
  float lam;
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, nkg, G, ngroups;
  int BR, nbands, nitems, WL;
  int pitch, rs_floats;
  int b_bytes;           // one of hi / lo: 2 K-atoms x Npad rows x 128 B
  int plain;             // 1: z <- c at every position (no z read, no step / shrinkage / mask / a3')
  int tau_stride;        // 0: tau[0] for every filter; 1: tau[k] per filter (ESO rule)
  int precise;           // plain mode: hi*hi and the cross terms in separate accumulators
  const int* sched;      // [G + 1] CTA offsets, then [nitems] items (code_h_schedule); nullptr: round robin
  unsigned long long* dbg;  // CSC_ROLE_TIMING: [grid][4 roles][8] cycle counters
  int dbgflags;             // CSC_ROLE_TIMING builds: CSC_CH_DBG experiment switches
};

struct ChItem {
  int n, u0, u1, p0, p1, ntiles, band;
};
// j: a position in the item list (the schedule's list, or the item itself without one)
__device__ __forceinline__ ChItem ch_item(const ChArgs& A, int j) {
  const int item = A.sched != nullptr ? A.sched[A.G + 1 + j] : j;
  ChItem it;
  it.n = item / A.nbands;
  it.band = item - it.n * A.nbands;
  it.u0 = it.band * A.BR;
  it.u1 = min(it.u0 + A.BR, A.Hc);
  it.p0 = it.u0 * A.Wc;
  it.p1 = it.u1 * A.Wc;
  it.ntiles = (it.p1 - it.p0 + kChTile - 1) / kChTile;
  return it;
}

template <int S>
__global__ void __launch_bounds__(kChThreads, 1) code_h_kernel(const __grid_constant__ ChArgs A) {
  constexpr int S2 = S * S;
  constexpr int P = S - 1;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t a_full[kChNS], a_empty[kChNS], acc_full[2], acc_empty[2], dz_full[2];
  __shared__ __align__(8) uint64_t y_full, y_empty;
  __shared__ __align__(8) uint64_t zfull[kChEpiWarps][kChChunks];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t dmax_sh, dl1_sh, tmax_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  // this CTA's item-list positions: jbeg, jbeg + jstep, ... < jend
  const int jbeg = A.sched != nullptr ? A.sched[gi] : gi;
  const int jend = A.sched != nullptr ? A.sched[gi + 1] : A.nitems;
  const int jstep = A.sched != nullptr ? 1 : A.G;
  const bool plain = A.plain != 0;
  const bool a3p = !plain && A.part != nullptr;
  // plain mode (ADMM's D^T e) with separate hi*hi / cross accumulators, single-buffered (T3)
  const bool prec = plain && A.precise != 0;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  uint8_t* bh = sm;                                              // [2 K-atoms][Npad][128 B] fp16 hi
  uint8_t* bl = sm + A.b_bytes;                                  // lo
  float* zsm = reinterpret_cast<float*>(sm + 2 * A.b_bytes);     // [16 warps][2][16][32]
  uint32_t* wsm = reinterpret_cast<uint32_t*>(zsm + kChEpiWarps * kZBuf);  // [epilogue warps][chunks][32]
  float* rs = reinterpret_cast<float*>(wsm + kChEpiWarps * kWBuf);  // residual pairs hi | lo [BR+P][pitch]
  float* win = rs + 2 * A.rs_floats;                             // [WL] band window of the a3' col2im

  // ---- setup: max|d|, max ||d_k||_1 and max tau of this filter group, then the fp16 hi/lo B image
  if (tid == 0) {
    dmax_sh = 0u;
    dl1_sh = 0u;
    tmax_sh = 0u;
  }
  for (int e = tid; e < A.WL; e += kChThreads) win[e] = 0.f;
  __syncthreads();
  {
    uint32_t m = 0u;
    for (int e = tid; e < A.KC * S2; e += kChThreads) {
      const int kk = kg * A.KC + e / S2;
      if (kk < A.K) m = max(m, __float_as_uint(fabsf(A.d[static_cast<size_t>(kg) * A.KC * S2 + e])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFullMask, m, o));
    if (lane == 0) atomicMax(&dmax_sh, m);
    if (!plain) {
      // one warp per filter: lanes sum strided taps, a shuffle tree finishes (fp32 sums: a bound only)
      for (int k = warp; k < A.KC; k += kChWarps) {
        const int kk = kg * A.KC + k;
        if (kk >= A.K) break;
        float l1 = 0.f;
        for (int t = lane; t < S2; t += 32) l1 += fabsf(A.d[static_cast<size_t>(kk) * S2 + t]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(kFullMask, l1, o);
        if (lane == 0) {
          atomicMax(&dl1_sh, __float_as_uint(l1 * 1.0001f));
          atomicMax(&tmax_sh, __float_as_uint(fabsf(A.tau[A.tau_stride ? kk : 0])));
        }
      }
    }
  }
  __syncthreads();
  const int ed = scale_exp_h(dmax_sh), er = scale_exp_h(*A.rmax);
  {
    const float sd = exp2i_h(ed);
    for (int e = tid; e < A.Npad * 64; e += kChThreads) {  // one thread per (k, tap pair)
      const int k = e >> 6, t = (e & 63) * 2;
      const int kk = kg * A.KC + k;
      const bool kok = k < A.KC && kk < A.K;
      const float v0 = (kok && t < S2) ? A.d[static_cast<size_t>(kk) * S2 + t] * sd : 0.f;
      const float v1 = (kok && t + 1 < S2) ? A.d[static_cast<size_t>(kk) * S2 + t + 1] * sd : 0.f;
      const float h0 = rn11_h(v0), h1 = rn11_h(v1);
      const int ka = t >> 6, w = t & 63;  // element w of 64 in the K-atom row
      const uint32_t off = static_cast<uint32_t>(ka * A.Npad * 128 + k * 128 + ((((w >> 3) ^ (k & 7))) << 4) + (w & 7) * 2);
      *reinterpret_cast<uint32_t*>(bh + off) = pack_h2_h(h0, h1);
      *reinterpret_cast<uint32_t*>(bl + off) = pack_h2_h(v0 - h0, v1 - h1);
    }
  }
  // |dz| <= tau (|c| + lambda) with |c| <= ||d_k||_1 max|r|  (a bound; only its exponent is used)
  const float dzb = plain ? 0.f
                          : __uint_as_float(tmax_sh) *
                                (__uint_as_float(dl1_sh) * __uint_as_float(*A.rmax) * 1.0001f + A.lam);
  const int edz = scale_exp_h(__float_as_uint(dzb));
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kChNS; ++i) {
      mbar_init(&a_full[i], kChHelpWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], a3p ? 1 : kChEpiWarps);  // a3': released by the GEMM 2 commit
      mbar_init(&dz_full[i], kChEpiWarps);
    }
    mbar_init(&y_full, 1);
    mbar_init(&y_empty, kChHelpWarps);
    for (int w = 0; w < kChEpiWarps; ++w)
      for (int c = 0; c < kChChunks; ++c) mbar_init(&zfull[w][c], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  if (warp == kChEpiBase && lane == 0 && !plain) {
    tma_prefetch_desc(&A.tm_z);
    if (A.mask != nullptr) tma_prefetch_desc(&A.tm_w);
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  const uint32_t t_acc = tbase;          // 2 x Npad columns
  const uint32_t t_a = tbase + kColA;    // kChNS slots x 64 columns
  const uint32_t t_y = tbase + kColY;    // 128 columns

  if (warp == 0) {
    // ================================ MMA issuer
    RoleClock rc;
    const uint32_t idesc = idesc_f16_kk(128, A.Npad);
    const uint32_t idesc2 = idesc_f16_kmn(128, 128);
    const uint32_t sbh = su32(bh), sbl = su32(bl);
    const uint32_t katom = static_cast<uint32_t>(A.Npad) * 128u;
    // GEMM 2 of tile u: Y = dz(u) x B (B read MN-major: taps contiguous, filters = K rows)
    auto gemm2 = [&](uint32_t u) {
      const uint32_t bu = u & 1u;
      RT_WAIT(rc, 2, mbar_wait_sleep(&dz_full[bu], (u >> 1) & 1u));
      RT_WAIT(rc, 3, mbar_wait_sleep(&y_empty, (u & 1u) ^ 1u));
      tc_after();
      const uint32_t acol = t_acc + bu * static_cast<uint32_t>(A.Npad);
      for (int c = 0; c < A.ngroups; ++c) {
        const uint64_t dbh = sdesc(sbh + static_cast<uint32_t>(c) * 2048u, katom, 1024u, kLayout128B);
        const uint64_t dbl = sdesc(sbl + static_cast<uint32_t>(c) * 2048u, katom, 1024u, kLayout128B);
        const uint32_t acc0 = c > 0 ? 1u : 0u;
        const uint32_t ah = acol + 16u * c;
        asm volatile(
            "{\n.reg .pred e, p, t;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %4, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %6, %4, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %4, t;\n"
            "}\n" ::"r"(t_y),
            "r"(ah), "r"(ah + 8u), "l"(dbh), "r"(idesc2), "r"(acc0), "l"(dbl)
            : "memory");
      }
      mma_commit_elect(&y_full);
      mma_commit_elect(&acc_empty[bu]);
    };
    uint32_t g = 0, tcount = 0;
    for (int item = jbeg; item < jend; item += jstep) {
      const ChItem it = ch_item(A, item);
      for (int tl = 0; tl < it.ntiles; ++tl, ++tcount) {
        const uint32_t buf = prec ? 0u : (tcount & 1u), use = prec ? tcount : (tcount >> 1);
        RT_WAIT(rc, 0, mbar_wait_sleep(&acc_empty[buf], (use & 1u) ^ 1u));
        tc_after();
        const uint32_t dcol = t_acc + buf * static_cast<uint32_t>(A.Npad);
        const uint32_t dxc = prec ? dcol + static_cast<uint32_t>(A.Npad) : dcol;  // cross-term accumulator
        for (int j = 0; j < 2; ++j, ++g) {  // 2 slots of 4 K16-steps (64 taps)
          const uint32_t slot = g % kChNS, ph = (g / kChNS) & 1u;
          RT_WAIT(rc, 1, mbar_wait_sleep(&a_full[slot], ph));
          tc_after();
          const uint32_t ah = t_a + slot * 64u;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // K16-step 4j + e: K-atom j, 32 B (16 fp16) into the 128-B row
            const uint64_t dbh = sdesc(sbh + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint64_t dbl = sdesc(sbl + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint32_t acc0 = (j > 0 || e > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred e, p, t, x;\n"
                "elect.sync _|e, 0xffffffff;\n"
                "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\nsetp.ne.b32 x, %8, 0;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %4, p;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%7], [%1], %6, %4, x;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%7], [%2], %3, %4, t;\n"
                "}\n" ::"r"(dcol),
                "r"(ah + 8u * e), "r"(ah + 32u + 8u * e), "l"(dbh), "r"(idesc), "r"(acc0), "l"(dbl), "r"(dxc),
                "r"(prec ? acc0 : 1u)
                : "memory");
          }
          mma_commit_elect(&a_empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
        if (a3p && tcount > 0) gemm2(tcount - 1);
      }
    }
    if (a3p && tcount > 0) gemm2(tcount - 1);
    __syncwarp();
    if (lane == 0) RT_DUMP(rc, A.dbg, 0);
  } else if (warp < kChHelpBase) {
    // ================================ epilogue: z <- S(z - tau c) on masked codes, dz -> TMEM
    const int ew = warp - kChEpiBase;  // 0..15
    const int q = warp & 3;
    const int jq = ew >> 2;            // 0..kChEpiPerQ-1: group rotation slot
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const float tau = plain ? 0.f : *A.tau;
    const float kappa = tau * A.lam;
    const float inv = exp2i_h(-(er + ed));
    const float ntinv = -tau * inv;
    const float sdz = exp2i_h(edz);
    const size_t plane = static_cast<size_t>(A.Hc) * A.Wc;
    const uint32_t planeB = static_cast<uint32_t>(plane * 4);  // < 2^28 for every supported shape: 16 planeB < 2^32
    const int kbase = kg * A.KC;
    const int kend = min(kbase + A.KC, A.K);
    const bool masked = A.mask != nullptr;
    float* zs0 = zsm + ew * kZBuf;     // [chunks][16 filters][32 positions]
    uint32_t* ws0 = wsm + ew * kWBuf;  // [chunks][32 positions] selection words
    // bits of the filters of group k0 .. k0+15 that exist (the rest of the group is padding)
    auto kvalid = [&](int k0) -> uint32_t {
      const int nv = kend - k0;
      return nv >= 16 ? 0xFFFFu : (nv <= 0 ? 0u : ((1u << nv) - 1u));
    };
    // tile cursors: the current tile and the next (its slices are loaded one tile ahead)
    int item = jbeg, tl = 0;
    ChItem it = ch_item(A, item < jend ? item : 0);
    int ni = item, ntl = 0;
    ChItem nit = it;
    auto step = [&](int& itm, int& t, ChItem& c) {
      if (++t >= c.ntiles) {
        t = 0;
        itm += jstep;
        if (itm < jend) c = ch_item(A, itm);
      }
    };
    // TMA of chunk s (group (jq + tc) mod E + E s, E = epilogue warps per quarter) of tile (itm, t): the {32 positions, 16 filters}
    // code slice and the 32 selection words; an empty arrival when the group does not exist
    auto issue = [&](int itm, int t, const ChItem& c, uint32_t tc, int s) {
      if (plain || itm >= jend) return;
      const int g = static_cast<int>((jq + tc) % kChEpiPerQ) + kChEpiPerQ * s;
      if (lane == 0) {
        if (g < A.ngroups) {
          const int pw = c.p0 + t * kChTile + 32 * q;
          mbar_arrive_expect_tx(&zfull[ew][s], 2048u + (masked ? 128u : 0u));
          tma_load_2d(su32(zs0 + s * 512), &A.tm_z, pw, c.n * A.K + kbase + 16 * g, &zfull[ew][s]);
          if (masked) tma_load_2d(su32(ws0 + s * 32), &A.tm_w, pw, kg * A.ngroups + g, &zfull[ew][s]);
        } else {
          mbar_arrive(&zfull[ew][s]);
        }
      }
    };
    float wmax = 0.f;
    RoleClock rc;
    uint32_t tcount = 0;
    for (int s0 = 0; s0 < kChChunks; ++s0) issue(item, tl, it, 0u, s0);
    if (ni < jend) step(ni, ntl, nit);
    while (item < jend) {
      const uint32_t buf = prec ? 0u : (tcount & 1u), use = prec ? tcount : (tcount >> 1);
      const int p = it.p0 + tl * kChTile + 32 * q + lane;
      const bool pok = p < it.p1;
      const int ga = static_cast<int>((jq + tcount) % kChEpiPerQ);
      RT_WAIT(rc, 0, mbar_wait_sleep(&acc_full[buf], use & 1u));
      tc_after();
      const uint32_t colb = t_acc + buf * static_cast<uint32_t>(A.Npad);
      float* zrow = A.z + (static_cast<size_t>(it.n) * A.K + kbase) * plane + p;
#pragma unroll 1
      for (int s = 0; s < kChChunks; ++s) {
        const int gg = ga + kChEpiPerQ * s;
        if (gg >= A.ngroups) {
          if (!plain) {
            RT_WAIT(rc, 1, mbar_wait_sleep(&zfull[ew][s], tcount & 1u));
            __syncwarp();
            issue(ni, ntl, nit, tcount + 1, s);
          }
          continue;
        }
        const int k0 = kbase + 16 * gg;
        const uint32_t kv = kvalid(k0);
        float c[16];
#ifdef CSC_ROLE_TIMING
        if (A.dbgflags & 2) {
#pragma unroll
          for (int i = 0; i < 16; ++i) c[i] = 0.f;
        } else
#endif
        {
          float c8[8];
          tmem_ld8_nowait(tq + colb + 16u * gg, c8);
#pragma unroll
          for (int i = 0; i < 8; ++i) c[i] = c8[i];
          tmem_ld8_nowait(tq + colb + 16u * gg + 8u, c8);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) c[8 + i] = c8[i];
          if (prec) {  // + the cross-term accumulator (fp32 add, round to nearest)
            const uint32_t cx = colb + static_cast<uint32_t>(A.Npad) + 16u * gg;
            tmem_ld8_nowait(tq + cx, c8);
#pragma unroll
            for (int i = 0; i < 8; ++i) c[i] += c8[i];
            tmem_ld8_nowait(tq + cx + 8u, c8);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) c[8 + i] += c8[i];
          }
        }
        float* zb = zrow + static_cast<size_t>(16 * gg) * plane;
        if (plain) {
          const uint32_t pv = pok ? kv : 0u;
#pragma unroll
          for (int i = 0; i < 16; ++i) st_global_if(zb + static_cast<size_t>(i) * plane, c[i] * inv, (pv >> i) & 1u);
          continue;
        }
        RT_WAIT(rc, 1, mbar_wait_sleep(&zfull[ew][s], tcount & 1u));
        const uint32_t wb = (masked ? ws0[s * 32 + lane] : 0xFFFFu) & (pok ? kv : 0u);
        float zc[16];
        const float* zr = zs0 + s * 512 + lane;
#pragma unroll
        for (int i = 0; i < 16; ++i) zc[i] = zr[32 * i];
        fence_async_shared();  // generic reads of the slice before the async-proxy refill
        __syncwarp();
        issue(ni, ntl, nit, tcount + 1, s);  // refill the chunk with the next tile's slice
        uint32_t hv[8], lv[8];
        // filters past the group's end are padding (K = 100: 4 of the last group's 16 are real)
        const int npair = kv == 0xFFFFu ? 8 : (32 - __clz(kv) + 1) >> 1;
        auto body = [&](auto per_k) {
          constexpr bool PK = decltype(per_k)::value;
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) {
            if (i2 >= npair) {  // warp-uniform
              hv[i2] = 0u;
              lv[i2] = 0u;
              continue;
            }
            const int i = 2 * i2;
            // -tau * (c * 2^-(er+ed)) with one multiply: scaling by a power of two is exact; the pair of
            // codes goes through the packed fp32 pipe (FFMA2 / FADD2 / FMUL2, each lane exact fp32)
            float tk0 = tau, tk1 = tau, kk0 = kappa, kk1 = kappa;
            if (PK) {
              tk0 = __ldg(A.tau + min(k0 + i, A.K - 1));
              tk1 = __ldg(A.tau + min(k0 + i + 1, A.K - 1));
              kk0 = tk0 * A.lam;
              kk1 = tk1 * A.lam;
            }
            const float2 zc2 = make_float2(zc[i], zc[i + 1]);
            const float2 w = __ffma2_rn(PK ? make_float2(-tk0 * inv, -tk1 * inv) : make_float2(ntinv, ntinv),
                                        make_float2(c[i], c[i + 1]), zc2);
            const float2 cl = make_float2(fminf(fmaxf(w.x, -kk0), kk0), fminf(fmaxf(w.y, -kk1), kk1));
            const float2 nz = __fadd2_rn(w, make_float2(-cl.x, -cl.y));  // S_kk(w): w -/+ kk outside, +0 inside
            // z_new - z_old on the selected codes, 0 elsewhere; a code changes iff its difference is
            // nonzero (x - y == 0 iff x == y in IEEE arithmetic with gradual underflow)
            const float2 dd = __fadd2_rn(nz, make_float2(-zc2.x, -zc2.y));
            const float2 dsel = make_float2((wb & (1u << i)) != 0u ? dd.x : 0.f, (wb & (2u << i)) != 0u ? dd.y : 0.f);
            // filter rows i, i + 1 of the slice: uniform byte offsets i * plane * 4 (< 2^32) from the slice base
            st_off_if_nz(zb, static_cast<uint32_t>(i) * planeB, nz.x, dsel.x);
            st_off_if_nz(zb, static_cast<uint32_t>(i + 1) * planeB, nz.y, dsel.y);
            // max |z| bound: every code of the slice was loaded, so |S(z - tau c)| over all of them bounds
            // the changed codes and the unchanged ones keep the previous bound
            wmax = fmaxf(wmax, fmaxf(fabsf(nz.x), fabsf(nz.y)));
            // dz split: hi = fp16_rn(dz_s), lo = fp16_rn(dz_s - hi) (dz_s - hi exact in fp32; T6)
            const float2 dz = __fmul2_rn(dsel, make_float2(sdz, sdz));
            const __half2 h2 = __float22half2_rn(dz);
            const float2 lo = __ffma2_rn(__half22float2(h2), make_float2(-1.f, -1.f), dz);
            const __half2 l2 = __float22half2_rn(lo);
            hv[i2] = *reinterpret_cast<const uint32_t*>(&h2);
            lv[i2] = *reinterpret_cast<const uint32_t*>(&l2);
          }
        };
#ifdef CSC_ROLE_TIMING
        if (A.dbgflags & 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) hv[i] = lv[i] = __float_as_uint(c[i] * zc[i]);
        } else
#endif
        if (A.tau_stride) body(std::true_type{});
        else body(std::false_type{});
        if (a3p) {
          tmem_st8(tq + colb + 16u * gg, hv);
          tmem_st8(tq + colb + 16u * gg + 8u, lv);
        }
      }
      if (a3p) {
        tmem_st_wait();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dz_full[buf]);
      } else {
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
      step(item, tl, it);
      if (ni < jend) step(ni, ntl, nit);
      ++tcount;
    }
    if (ew == 0 && lane == 0) RT_DUMP(rc, A.dbg, 2);
    uint32_t wbm = __float_as_uint(wmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wbm = max(wbm, __shfl_xor_sync(kFullMask, wbm, o));
    if (lane == 0 && A.zmax != nullptr && wbm != 0u) atomicMax(A.zmax, wbm);
  } else {
    // ================================ helpers (8 = 4 TMEM lane quarters x 2): per tile t, the im2col of
    // tile t (their half of each slot's K16-steps), then the col2im of tile t-1 (their half of the tap rows)
    const int q = warp & 3;
    const int hh = (warp - kChHelpBase) >> 2;  // 0, 1
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const int ht = tid - 32 * kChHelpBase;     // 0..255
    const float sr = exp2i_h(er);
    RoleClock rc;
    // The band's residual rows u0-P .. u1-1 (columns -P .. Wc-1, zero outside the image), scaled by
    // 2^er and split once per band into fp16 hi / lo PAIRS: hp[row][c] = (hi(r[row][c-P]), hi(r[row][c-P+1])),
    // lp likewise.  A TMEM column of the im2col holds two consecutive taps (a, b), (a, b+1) of one
    // position, which is then a single 32-bit shared load of each array (no per-tap arithmetic).
    uint32_t* hp = reinterpret_cast<uint32_t*>(rs);
    uint32_t* lp = hp + A.rs_floats;
    auto fill = [&](const ChItem& it) {
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      for (int e = ht; e < A.rs_floats; e += 32 * kChHelpWarps) {
        const int rho = e / A.pitch, c = e - rho * A.pitch;
        const int i = it.u0 - P + rho, jj = c - P;
        const bool iok = i >= 0 && i < A.H;
        const float* rr = rn + static_cast<size_t>(iok ? i : 0) * A.W;
        const float x0 = (iok && jj >= 0 && jj < A.W) ? __ldg(rr + jj) * sr : 0.f;
        const float x1 = (iok && jj + 1 >= 0 && jj + 1 < A.W) ? __ldg(rr + jj + 1) * sr : 0.f;
        const float h0 = rn11_h(x0), h1 = rn11_h(x1);
        hp[e] = pack_h2_h(h0, h1);
        lp[e] = pack_h2_h(x0 - h0, x1 - h1);
      }
    };
    // im2col of tile (it, tl), count tc: for each slot j, this warp's K16-steps 2 hh, 2 hh + 1
    auto convert = [&](const ChItem& it, int tl, uint32_t tc) {
      const int p = it.p0 + tl * kChTile + 32 * q + lane;
      const bool pok = p < it.p1;
      const int u = p / A.Wc, v = p - u * A.Wc;
      const int o = pok ? (u - it.u0) * A.pitch + v : 0;
      const uint32_t* sh = hp + o;
      const uint32_t* sl = lp + o;
#pragma unroll
      for (int j = 0; j < 2; ++j) {  // slot j: taps 64 j .. 64 j + 63
        RT_WAIT(rc, 1, mbar_wait_sleep(&a_empty[j], (tc & 1u) ^ 1u));
        tc_after();
        auto cols = [&](auto ec) {
          constexpr int E0 = decltype(ec)::value;
#pragma unroll
          for (int ee = 0; ee < 2; ++ee) {
            const int e = E0 + ee;  // K16-step within the slot
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int t0 = 64 * j + 16 * e + 2 * jj, t1 = t0 + 1;
              const int a0 = t0 / S, b0 = t0 % S, a1 = t1 / S, b1 = t1 % S;
              uint32_t xh = 0u, xl = 0u;
              if (t0 < S2) {
                const int o0 = a0 * A.pitch + b0;
                if (t1 < S2 && a1 == a0) {  // both taps in one row: the stored pair
                  xh = sh[o0];
                  xl = sl[o0];
                } else {                     // the pair straddles two tap rows (or ends the taps)
                  const uint32_t h0 = sh[o0], l0 = sl[o0];
                  if (t1 < S2) {
                    const int o1 = a1 * A.pitch + b1;
                    xh = __byte_perm(h0, sh[o1], 0x5410);
                    xl = __byte_perm(l0, sl[o1], 0x5410);
                  } else {
                    xh = h0 & 0xFFFFu;
                    xl = l0 & 0xFFFFu;
                  }
                }
              }
              hv[jj] = pok ? xh : 0u;
              lv[jj] = pok ? xl : 0u;
            }
            const uint32_t col = t_a + j * 64u + 8u * e;
            tmem_st8(tq + col, hv);
            tmem_st8(tq + col + 32u, lv);
          }
        };
        if (hh == 0) cols(std::integral_constant<int, 0>{});
        else cols(std::integral_constant<int, 2>{});
        tmem_st_wait();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[j]);
      }
    };
    // col2im of Y of tile (it, t), count tc, into the band window
    constexpr int AH = (S + 1) / 2;
    const int a0 = hh * AH, a1 = hh ? S : AH;
    float hm[S];  // [lane < b]: the rotations of tap b that belong to the next quarter (col2im halo)
#pragma unroll
    for (int b = 0; b < S; ++b) hm[b] = lane < b ? 1.f : 0.f;
    const float inv2 = exp2i_h(-(edz + ed));
    // add phases: the quarters in order (and the two row halves of a quarter in order when their windows
    // can overlap, Wc < 32 + P): deterministic fp32 sums
    const bool wide = A.Wc >= kChTile;
    const bool split = A.Wc < 32 + P;
    const int nph = split ? 8 : 4;
    const int myph = split ? 2 * q + hh : q;
    auto col2im = [&](const ChItem& it, int t, uint32_t tc) {
      RT_WAIT(rc, 0, mbar_wait_sleep(&y_full, tc & 1u));
      tc_after();
      const int pq = 128 * t + 32 * q;
      const bool pvalid = it.p0 + pq + lane < it.p1;
      const uint32_t tacc = t_y + (static_cast<uint32_t>(32 * q) << 16);
      float* rowb = win + pq + lane;
      float own[AH], dnv[AH];
      // two tap rows at a time through the packed fp32 pipe: one rotation per tap serves both parts (lanes
      // >= b get position lane-b of this quarter, lanes < b position lane-b+32, the halo of the next quarter's
      // first lanes); tot sums every rotation, hal the halo ones (x hm[b] = [lane < b], exact), own = tot - hal
      auto rows = [&](auto partial) {
        constexpr bool PART = decltype(partial)::value;
#pragma unroll
        for (int i = 0; i < AH; i += 2) {
          own[i] = dnv[i] = 0.f;
          if (i + 1 < AH) own[i + 1] = dnv[i + 1] = 0.f;
          const int a = a0 + i;
          if (a >= a1) continue;
          const bool two = i + 1 < AH && a + 1 < a1;  // warp-uniform
          float y0[S], y1[S];
          tmem_ld_row<S>(tacc + a * S, y0);
          if (two) tmem_ld_row<S>(tacc + (a + 1) * S, y1);
          tmem_ld_wait();
          float2 tot = make_float2(0.f, 0.f), hal = make_float2(0.f, 0.f);
#pragma unroll
          for (int b = 0; b < S; ++b) {
            const float v0 = PART ? (pvalid ? y0[b] : 0.f) : y0[b];
            const float v1 = two ? (PART ? (pvalid ? y1[b] : 0.f) : y1[b]) : 0.f;
            const float2 rot = b == 0 ? make_float2(v0, v1)
                                      : make_float2(__shfl_sync(kFullMask, v0, (lane - b) & 31),
                                                    __shfl_sync(kFullMask, v1, (lane - b) & 31));
            tot = __fadd2_rn(tot, rot);
            if (b > 0) hal = __ffma2_rn(rot, make_float2(hm[b], hm[b]), hal);
          }
          own[i] = tot.x - hal.x;
          dnv[i] = hal.x;
          if (i + 1 < AH) {
            own[i + 1] = tot.y - hal.y;
            dnv[i + 1] = hal.y;
          }
        }
      };
      if (__all_sync(kFullMask, pvalid)) rows(std::false_type{});
      else rows(std::true_type{});
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&y_empty);
      if (wide) {
        // Wc >= 128: the own values of all quarters and tap-row halves hit distinct window cells, and so do
        // the halo values; two phases (own, then halo) keep every cell's sum in a fixed order
#pragma unroll
        for (int i = 0; i < AH; ++i)
          if (a0 + i < a1) rowb[(a0 + i) * A.Wc] += own[i];
        RT_WAIT(rc, 2, named_sync(2, 32 * kChHelpWarps));
        if (lane < P) {
#pragma unroll
          for (int i = 0; i < AH; ++i)
            if (a0 + i < a1) rowb[(a0 + i) * A.Wc + 32] += dnv[i];
        }
        RT_WAIT(rc, 2, named_sync(2, 32 * kChHelpWarps));
        return;
      }
#pragma unroll 1
      for (int ph = 0; ph < nph; ++ph) {
        if (ph == myph) {
#pragma unroll
          for (int i = 0; i < AH; ++i)
            if (a0 + i < a1) rowb[(a0 + i) * A.Wc] += own[i];
          __syncwarp();
          if (lane < P) {
#pragma unroll
            for (int i = 0; i < AH; ++i)
              if (a0 + i < a1) rowb[(a0 + i) * A.Wc + 32] += dnv[i];
          }
        }
        RT_WAIT(rc, 2, named_sync(2, 32 * kChHelpWarps));
      }
    };
    // flush the band window: output rows u0-P .. u0+BR-1 (window row r = output row u0-P+r)
    auto flush = [&](const ChItem& it) {
      float* dst = A.part + ((static_cast<size_t>(kg) * A.N + it.n) * A.nbands + it.band) *
                                static_cast<size_t>(A.BR + P) * A.W;
      const int nrows = A.BR + P;
      for (int e = ht; e < nrows * A.W; e += 32 * kChHelpWarps) {
        const int r = e / A.W, jc = e - r * A.W;
        dst[e] = win[r * A.Wc + jc + P] * inv2;  // exact: power of two
      }
      named_sync(2, 32 * kChHelpWarps);
      for (int e = ht; e < A.WL; e += 32 * kChHelpWarps) win[e] = 0.f;
      named_sync(2, 32 * kChHelpWarps);
    };
    // per tile t: the im2col of tile t+1 (the tensor pipe needs it right after C(t)), then the col2im of
    // tile t-1 (its Y is ready once GEMM 2 of t-1, issued after C(t), completes)
    int item = jbeg;
    if (item < jend) {
      ChItem it = ch_item(A, item);
      int tl = 0;
      ChItem pit = it;
      int ptl = 0;
      int nitem = item, ntl = 0;
      ChItem nit = it;
      auto step = [&](int& itm, int& t, ChItem& c) {
        if (++t >= c.ntiles) {
          t = 0;
          itm += jstep;
          if (itm < jend) c = ch_item(A, itm);
        }
      };
      fill(it);
      RT_WAIT(rc, 3, named_sync(1, 32 * kChHelpWarps));
      convert(it, 0, 0u);
      step(nitem, ntl, nit);
      uint32_t tcount = 0;
      while (item < jend) {
        if (nitem < jend) {
          if (nitem != item) {  // a new band: every helper is past its last use of the residual pairs
            RT_WAIT(rc, 3, named_sync(1, 32 * kChHelpWarps));
            fill(nit);
            RT_WAIT(rc, 3, named_sync(1, 32 * kChHelpWarps));
          }
          convert(nit, ntl, tcount + 1);
        }
        if (a3p && tcount > 0) {
          col2im(pit, ptl, tcount - 1);
          if (ptl == pit.ntiles - 1) flush(pit);
        }
        pit = it;
        ptl = tl;
        item = nitem;
        tl = ntl;
        it = nit;
        if (nitem < jend) step(nitem, ntl, nit);
        ++tcount;
      }
      if (a3p && tcount > 0) {
        col2im(pit, ptl, tcount - 1);
        flush(pit);
      }
    }
    if (warp == kChHelpBase && lane == 0) RT_DUMP(rc, A.dbg, 1);
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// r += sum_kg sum_{bands b covering row i} part[kg][n][b][i - b BR + P][j]  (fixed order)
__global__ void code_a3_fixup_kernel(const float* __restrict__ part, int nkg, int N, int H, int W, int P, int BR,
                                     int nbands, float* __restrict__ r) {
  const size_t win = static_cast<size_t>(BR + P) * W;
  const size_t kstride = static_cast<size_t>(N) * nbands * win;
  const int64_t total = static_cast<int64_t>(N) * H * W;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / W;
    const int j = static_cast<int>(e - row * W);
    const int n = static_cast<int>(row / H), i = static_cast<int>(row - static_cast<int64_t>(n) * H);
    const int b0 = i / BR;
    int b1 = (i + P) / BR;
    if (b1 > nbands - 1) b1 = nbands - 1;
    float v = 0.f;
    for (int kg = 0; kg < nkg; ++kg) {
      const float* pk = part + kg * kstride + static_cast<size_t>(n) * nbands * win;
      for (int b = b0; b <= b1; ++b) v += pk[b * win + static_cast<size_t>(i - b * BR + P) * W + j];
    }
    r[e] += v;
  }
}

// the same with 4 columns per thread (W % 4 == 0, 16-B aligned buffers): one float4 per band partial
__global__ void code_a3_fixup4_kernel(const float4* __restrict__ part, int nkg, int N, int H, int W4, int P, int BR,
                                      int nbands, float4* __restrict__ r) {
  const size_t win4 = static_cast<size_t>(BR + P) * W4;
  const size_t kstride4 = static_cast<size_t>(N) * nbands * win4;
  const int total = N * H * W4;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int row = e / W4, j4 = e - row * W4;
    const int n = row / H, i = row - n * H;
    const int b0 = i / BR;
    int b1 = (i + P) / BR;
    if (b1 > nbands - 1) b1 = nbands - 1;
    float4 v = r[e];
    for (int kg = 0; kg < nkg; ++kg) {
      const float4* pk = part + kg * kstride4 + static_cast<size_t>(n) * nbands * win4;
      for (int b = b0; b <= b1; ++b) {
        const float4 t = __ldg(pk + b * win4 + static_cast<size_t>(i - b * BR + P) * W4 + j4);
        v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w;
      }
    }
    r[e] = v;
  }
}

template <int S>
cudaError_t run_code_h(const ChArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&code_h_kernel<S>), kChSmemMax);
  if (e != cudaSuccess) return e;
#ifdef CSC_ROLE_TIMING
  static unsigned long long* dbg = nullptr;
  static int calls = 0;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 32 * 1024);
  cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 32 * 1024, st);
  ChArgs b = a;
  b.dbg = dbg;
  b.dbgflags = std::getenv("CSC_CH_DBG") ? std::atoi(std::getenv("CSC_CH_DBG")) : 0;
  code_h_kernel<S><<<grid, kChThreads, smem, st>>>(b);
  if (++calls % 4 == 0) {
    static unsigned long long h[32 * 1024];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(unsigned long long) * 32 * grid, cudaMemcpyDeviceToHost);
    double t[32] = {0};
    for (int bk = 0; bk < grid; ++bk)
      for (int i = 0; i < 32; ++i) t[i] += static_cast<double>(h[bk * 32 + i]) / grid;
    fprintf(stderr,
            "[code_h roles] mma: total %.0f w_accempty %.0f w_afull %.0f w_dzfull %.0f w_yempty %.0f | helper: total "
            "%.0f w_yfull %.0f w_aempty %.0f w_phase %.0f w_fill %.0f | epi: total %.0f w_accfull %.0f w_zfull %.0f\n",
            t[7], t[0], t[1], t[2], t[3], t[15], t[8], t[9], t[10], t[11], t[23], t[16], t[17]);
  }
#else
  code_h_kernel<S><<<grid, kChThreads, smem, st>>>(a);
#endif
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- host side
bool code_h_supported(const Geom& g) {
  // TMA views of z and of the selection words: rows of Hc*Wc elements must be 16-byte multiples
  return g.N > 0 && (g.S == 3 || g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) &&
         (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 && tmap_available();
}

CodeTcPlan code_h_plan(const Geom& g, int num_sms) {
  CodeTcPlan p{};
  p.nkg = ceil_div(g.K, 112);
  p.KC = ceil_div(g.K, p.nkg);
  p.Npad = (p.KC + 15) / 16 * 16;
  p.ngroups = p.Npad / 16;
  p.wnc = 16;
  p.wper = p.ngroups;
  p.b_bytes = 2 * p.Npad * 128;
  int pitch = g.Wc + g.P;
  while (pitch % 32 != 0) ++pitch;
  p.pitch = pitch;
  const int plane = g.Hc * g.Wc;
  p.sw_words = static_cast<size_t>(p.nkg) * p.ngroups * plane;
  const int G = num_sms / p.nkg > 0 ? num_sms / p.nkg : 1;
  const int n = g.N > 0 ? g.N : 1;
  const int smem_fixed = 1024 + 2 * p.b_bytes + kChEpiWarps * (kZBuf + kWBuf) * 4;
  auto smem_for = [&](int br) {
    const int rs = (br + g.P) * pitch;
    const int wl = (br + g.P) * g.Wc + 192;
    return smem_fixed + 2 * rs * 4 + wl * 4;
  };
  // band height: the smallest busiest-CTA cost (128-position tiles + 2 per band for the residual staging and
  // the window flush) under the LPT schedule of code_h_schedule, the taller band on ties
  int best = 0;
  int64_t best_cost = 0;
  for (int br = 1; br <= 32 && br <= g.Hc; ++br) {
    if (smem_for(br) > kChSmemMax) break;
    if ((br * g.Wc) % 4 != 0) continue;  // every band starts 16-B aligned (TMA box starts)
    const int nb = ceil_div(g.Hc, br);
    const int64_t cost = g.N > 0 ? lpt_bands(g, br, std::min(G, n * nb), 2, nullptr) : br;
    if (best == 0 || cost <= best_cost) {
      best = br;
      best_cost = cost;
    }
  }
  if (best == 0) {
    p.ok = false;
    return p;
  }
  p.BR = best;
  p.nbands = ceil_div(g.Hc, p.BR);
  p.rs_rows = p.BR + g.P;
  p.rs_floats = p.rs_rows * pitch;
  p.WL = (p.BR + g.P) * g.Wc + 192;
  p.nitems = g.N * p.nbands;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_for(p.BR);
  p.a3_floats = static_cast<size_t>(p.nkg) * g.N * p.nbands * (p.BR + g.P) * g.W;
  p.ok = p.smem <= kChSmemMax;
  p.half = true;
  return p;
}

void code_h_schedule(const Geom& g, const CodeTcPlan& p, std::vector<int>& out) {
  if (g.N <= 0 || p.nitems <= 0) {
    out.assign(p.G + 1, 0);
    return;
  }
  lpt_bands(g, p.BR, p.G, 2, &out);
}

cudaError_t launch_code_h(const Geom& g, const CodeTcPlan& p, TmapCache* tmc, const float* r, const float* d,
                          float* z, const uint32_t* words, const float* tau_dev, float lam, const uint32_t* rmax,
                          uint32_t* zmax, cudaStream_t st, bool plain, int tau_stride, float* a3_part) {
  ChArgs a{};
  if (!plain) {
    const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
    cudaError_t e = tmap_2d(tmc[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K,
                            plane * 4, 32, 16, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    if (e != cudaSuccess) return e;
    a.tm_z = tmc[0].map;
    if (words != nullptr) {
      e = tmap_2d(tmc[1], CU_TENSOR_MAP_DATA_TYPE_UINT32, words, plane, static_cast<uint64_t>(p.nkg) * p.ngroups,
                  plane * 4, 32, 1, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
      if (e != cudaSuccess) return e;
      a.tm_w = tmc[1].map;
    }
  }
  a.r = r; a.d = d; a.z = z; a.mask = words; a.tau = tau_dev; a.lam = lam; a.rmax = rmax; a.zmax = zmax;
  a.part = plain ? nullptr : a3_part;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.Npad = p.Npad; a.nkg = p.nkg; a.G = p.G; a.ngroups = p.ngroups;
  a.BR = p.BR; a.nbands = p.nbands; a.nitems = p.nitems; a.WL = p.WL;
  a.pitch = p.pitch; a.rs_floats = p.rs_floats; a.b_bytes = p.b_bytes;
  a.plain = plain ? 1 : 0;
  a.precise = plain ? 1 : 0;  // the plain correlation (ADMM) always takes the precise accumulation
  a.tau_stride = tau_stride;
  a.sched = p.sched;
  if (plain) {
    a.mask = nullptr;
    a.zmax = nullptr;
  }
  switch (g.S) {
    case 3: return run_code_h<3>(a, p.grid, p.smem, st);
    case 5: return run_code_h<5>(a, p.grid, p.smem, st);
    case 7: return run_code_h<7>(a, p.grid, p.smem, st);
    case 9: return run_code_h<9>(a, p.grid, p.smem, st);
    case 11: return run_code_h<11>(a, p.grid, p.smem, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_code_a3_fixup(const Geom& g, const CodeTcPlan& p, const float* part, float* r, cudaStream_t st) {
  if (g.N == 0) return cudaSuccess;
  if (g.W % 4 == 0 && (reinterpret_cast<uintptr_t>(part) & 15u) == 0 && (reinterpret_cast<uintptr_t>(r) & 15u) == 0 &&
      static_cast<int64_t>(g.N) * g.H * (g.W / 4) < (int64_t(1) << 31)) {
    const int total = g.N * g.H * (g.W / 4);
    const int blocks = total / 256 + 1;  // one float4 per thread: every load in flight at once
    code_a3_fixup4_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(part), p.nkg, g.N, g.H, g.W / 4,
                                                   g.P, p.BR, p.nbands, reinterpret_cast<float4*>(r));
  } else {
    code_a3_fixup_kernel<<<kFinalizeBlocks, 256, 0, st>>>(part, p.nkg, g.N, g.H, g.W, g.P, p.BR, p.nbands, r);
  }
  return cudaGetLastError();
}

}  // namespace csc

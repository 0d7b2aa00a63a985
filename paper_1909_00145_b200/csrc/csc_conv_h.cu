// csc_conv_h.cu -- dense pass y = sum_k f_k * z_k on the sm_100a tensor cores, 3-term fp16 split
// (tcgen05.mma kind::f16, fp32 accumulate), TMA-fed shared-memory operands.
//
// Same mathematics and tiling as csc_conv_ss.cu: Y[pos][tap] =
// sum_k z[k][pos] f[k][tap] on flattened 128-position tiles, warp-shuffle col2im into one band
// window.  The operands are split into two fp16 halves after an exact power-of-two scaling
// (reading T6):
//   x_s = x * 2^e,  hi = rn11(x_s) (rounded to 11 significant bits in fp32, exactly an fp16),
//   lo = fp16_rn(x_s - hi),   Y_s += A_hi B_hi + A_hi B_lo + A_lo B_hi,   Y = Y_s * 2^-(e_z + e_f)
// which carries the same 2^-22 per-product error as the 3xTF32 split while the tensor core runs at
// the fp16 rate (2x tf32) with half the shared-memory bytes per MAC.  e_f comes from max|f|
// (computed by the B-image kernel), e_z from a running upper bound of max|z| that the code step
// raises whenever it writes a code (csc_api.cu keeps it); both put the largest scaled magnitude
// at <= 2^14, so no value overflows fp16 and values below 2^-24 of the maximum lose nothing that
// survives the fp32 sum.
//
// Stage = 16 filter planes of one tile: one TMA box {128 positions, 16 planes} (fp32, no swizzle,
// 8 KB: one request per stage keeps the TMA issue rate off the critical path) into a raw slot, converted
// by a pair of converter warps into fp16 hi/lo tiles in the canonical MN-major SWIZZLE_128B layout (2 atoms
// of 64 positions x 16 rows of 128 B, 16-B chunks XOR row); the raw slot is released once converted, the
// hi/lo slot once multiplied.
// CTA (persistent, 32 warps, <= 64 registers): warp 0 MMA, warp 1 TMA, warps 2..19 converters (a pair
// per slot), warps 20..31 epilogue (4 TMEM lane quarters x 3 groups of tap rows).  CSC_CH_NS / CSC_CH_NR /
// CSC_CH_EPI_GROUPS / CSC_CH_SPLIT_CVT change the split in tuning builds (A/B at config 3: 9 slots with the
// rn11 split 0.338 ms, with the cvt-based split 0.330; 7 slots and 4 epilogue groups 0.391; 5 / 5 0.457).
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <queue>
#include <type_traits>
#include <utility>
#include <vector>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

#ifndef CSC_CH_NS
#define CSC_CH_NS 9
#endif
#ifndef CSC_Z_EVICT_FIRST
#define CSC_Z_EVICT_FIRST 0  // evict-first z loads (tcx::tma_load_2d_hint): measured 0.333 -> 0.337 ms here, off
#endif
#ifndef CSC_CH_NR
#define CSC_CH_NR CSC_CH_NS
#endif
#ifndef CSC_CH_SPLIT_CVT
#define CSC_CH_SPLIT_CVT 1
#endif
#ifndef CSC_CH_EPI_GROUPS
#define CSC_CH_EPI_GROUPS 3
#endif
constexpr int kHNS = CSC_CH_NS;     // hi / lo slots (16 filters of one tile each)
constexpr int kHNR = CSC_CH_NR;     // raw fp32 slots (TMA boxes in flight); >= kHNS
// a raw slot's stages (g = r mod kHNR) must all go to one converter pair (g mod kHNS): a pair waits its
// slots' phases in order, so no waiter ever runs a full phase ahead of the barrier (parity aliasing)
static_assert(kHNR % kHNS == 0, "raw ring depth must be a multiple of the hi / lo ring depth");
constexpr int kHConvWarps = 2 * kHNS;  // 2 per hi / lo slot (kHNS slots): a slot is always converted by the same pair
constexpr int kHEpiGroups = CSC_CH_EPI_GROUPS;  // groups of tap rows
constexpr int kHEpiWarps = 4 * kHEpiGroups;     // 4 lane quarters x kHEpiGroups groups of tap rows
constexpr int kHConvBase = 2, kHEpiBase = kHConvBase + kHConvWarps;
constexpr int kHWarps = kHEpiBase + kHEpiWarps;
constexpr int kHThreads = 32 * kHWarps;
constexpr int kHRawBytes = 8192;    // one TMA box: 16 planes x 128 positions (fp32, rows of 512 B)
constexpr int kHHalfBytes = 4096;   // 2 atoms x 16 rows x 128 B (fp16), one of hi / lo
constexpr int kHRingBytes = kHNR * kHRawBytes + kHNS * 2 * kHHalfBytes;
constexpr int kHSmemMax = 226 * 1024;  // + the static smem stays under the 227 KB opt-in limit

// instruction descriptor kind::f16: fp32 accumulate, fp16 A/B, both MN-major
__host__ __device__ constexpr uint32_t idesc_f16_mn(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// scale exponent for a magnitude bound m (float bits): 2^e with m * 2^e <= 2^14
__device__ __forceinline__ int scale_exp(uint32_t mbits) {
  if ((mbits & 0x7FFFFFFFu) == 0u) return 0;
  const int E = static_cast<int>((mbits >> 23) & 0xFFu) - 127;  // m in [2^E, 2^(E+1))
  int e = 13 - E;                                                 // m * 2^e < 2^14
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}
__device__ __forceinline__ float exp2i(int e) { return __uint_as_float(static_cast<uint32_t>(e + 127) << 23); }

__device__ __forceinline__ float rn11(float x) {  // round to 11 significant bits (an fp16 mantissa)
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

#ifdef CSC_ROLE_TIMING
#define HT_NOW() clock64()
#else
#define HT_NOW() 0ull
#endif

struct HArgs {
  const uint16_t* bimg;      // [nks][2][2 atoms][KC][64] fp16, SW128
  const uint32_t* zmax;      // bound on max |z| (float bits)
  const uint32_t* fmax;      // max |f| (float bits), written by the B-image kernel
  float* part;               // [N][nbands][BR+P][W]
  double* l1_part;           // [nks * grid] or nullptr
  int N, K, S, H, W, Hc, Wc, P;
  int KC, NCH, NT, ks;       // NCH = KC / 16
  int BR, nbands, nitems, WL;
  int precise;  // 1: hi*hi and the cross terms in separate TMEM accumulators (the ||Zg||^2 pass, reading T3)
  const int* sched;  // [grid + 1] CTA offsets, then [nitems] items (conv_h_schedule); nullptr: round robin
  unsigned long long* dbg;  // CSC_ROLE_TIMING builds: per-CTA role cycle counters [grid][16]
};

struct HItem {
  int n, u0, u1, p0, pend, ntiles;
};
__device__ __forceinline__ HItem h_item(const HArgs& A, int item) {
  HItem it;
  it.n = item / A.nbands;
  const int b = item - it.n * A.nbands;
  it.u0 = b * A.BR;
  it.u1 = min(it.u0 + A.BR, A.Hc);
  it.p0 = it.u0 * A.Wc;
  it.pend = it.u1 * A.Wc;
  it.ntiles = (it.pend - it.p0 + 127) / 128;
  return it;
}

// the items of this CTA: positions j in [j0, j1) of its list (the balanced schedule of conv_h_schedule, or
// blockIdx.x + j * gridDim.x without one)
__device__ __forceinline__ void h_range(const HArgs& A, int& j0, int& j1) {
  if (A.sched != nullptr) {
    j0 = A.sched[blockIdx.x];
    j1 = A.sched[blockIdx.x + 1];
  } else {
    j0 = 0;
    j1 = A.nitems > static_cast<int>(blockIdx.x) ? (A.nitems - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1 : 0;
  }
}
__device__ __forceinline__ int h_item_at(const HArgs& A, int j) {
  return A.sched != nullptr ? A.sched[gridDim.x + 1 + j] : static_cast<int>(blockIdx.x) + j * gridDim.x;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

template <int S>
__global__ void __launch_bounds__(kHThreads, 1)
conv_h_kernel(const __grid_constant__ CUtensorMap tmap_z, const HArgs A) {
  constexpr int P = S - 1;
  extern __shared__ uint8_t smraw[];
  // per stage slot: full (TMA -> converters), rempty (converters done reading the raw tile -> TMA),
  // ready (hi / lo written -> MMA), empty (MMA done reading hi / lo -> converters)
  __shared__ __align__(8) uint64_t full[kHNR], rempty[kHNR], ready[kHNS], empty[kHNS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double l1_warp[kHConvWarps];

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int bbytes = 2 * A.KC * 128;                   // one of hi / lo: 2 atoms x KC rows x 128 B
  uint8_t* bsm = sm;                                   // [hi | lo]
  uint8_t* stg = sm + 2 * bbytes;                      // [NS][raw 8 KB | hi 4 KB | lo 4 KB]
  // stg = [kHNR raw slots of 8 KB][kHNS hi / lo slots of 8 KB]
  uint8_t* hls = stg + kHNR * kHRawBytes;
  float* win = reinterpret_cast<float*>(stg + kHRingBytes);  // [WL]
  const int ez = scale_exp(*A.zmax), ef = scale_exp(*A.fmax);

  {
    const int4* src = reinterpret_cast<const int4*>(A.bimg + static_cast<size_t>(A.ks) * 2 * 2 * A.KC * 64);
    int4* dst = reinterpret_cast<int4*>(bsm);
    for (int e = tid; e < 2 * bbytes / 16; e += kHThreads) dst[e] = src[e];
    for (int e = tid; e < A.WL; e += kHThreads) win[e] = 0.f;
  }
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kHNR; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&rempty[i], 2);
    }
    for (int i = 0; i < kHNS; ++i) {
      mbar_init(&ready[i], 2);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kHEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 1 && lane == 0) tma_prefetch_desc(&tmap_z);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  int j0, j1;
  h_range(A, j0, j1);

  if (warp == 0) {
    // ================================ MMA issuer
    const uint32_t idesc = idesc_f16_mn(128, A.NT);
    const uint32_t lbo_b = static_cast<uint32_t>(A.KC) * 128u;  // N atom (64 taps) stride
    const uint32_t sbh = su32(bsm), sbl = su32(bsm + bbytes), sst = su32(hls);
    uint32_t g = 0, tcount = 0;
    unsigned long long t0 = HT_NOW(), w_ae = 0, w_rd = 0;
    for (int j = j0; j < j1; ++j) {
      const int item = h_item_at(A, j);
      const HItem it = h_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        unsigned long long ta = HT_NOW();
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        w_ae += HT_NOW() - ta;
        tc_after();
        // accumulator buffer: 256 columns [hi*hi | cross terms] (precise) or 128 (one accumulator)
        const uint32_t d = tbase + buf * (A.precise ? 256u : 128u);
        const uint32_t dx = A.precise ? d + 128u : d;
        for (int c = 0; c < A.NCH; ++c, ++g) {
          const uint32_t slot = g % kHNS, ph = (g / kHNS) & 1u;
          unsigned long long tb = HT_NOW();
          mbar_wait(&ready[slot], ph);
          w_rd += HT_NOW() - tb;
          tc_after();
          const uint32_t ah = sst + slot * (2 * kHHalfBytes);
          // A: MN-major SW128, 2 atoms of 64 positions at LBO = 16 rows x 128 B, 8-row K groups at SBO
          const uint64_t dah = sdesc(ah, 2048u, 1024u, kLayout128B);
          const uint64_t dal = sdesc(ah + kHHalfBytes, 2048u, 1024u, kLayout128B);
          // B: K-step c = filter rows 16c..16c+15 of the resident image
          const uint64_t dbh = sdesc(sbh + static_cast<uint32_t>(c) * 2048u, lbo_b, 1024u, kLayout128B);
          const uint64_t dbl = sdesc(sbl + static_cast<uint32_t>(c) * 2048u, lbo_b, 1024u, kLayout128B);
          const uint32_t acc0 = c > 0 ? 1u : 0u;
          // precise: the cross terms start their own accumulator (flag p), so the tensor core's
          // accumulate rounding acts on the small cross sums, not on the hi*hi sum
          asm volatile(
              "{\n.reg .pred e, p, t, x;\n"
              "elect.sync _|e, 0xffffffff;\n"
              "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\nsetp.ne.b32 x, %8, 0;\n"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %4, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%7], %1, %6, %4, x;\n"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%7], %2, %3, %4, t;\n"
              "}\n" ::"r"(d),
              "l"(dah), "l"(dal), "l"(dbh), "r"(idesc), "r"(acc0), "l"(dbl), "r"(dx),
              "r"(A.precise ? acc0 : 1u)
              : "memory");
          mma_commit_elect(&empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    if (A.dbg && lane == 0) {
      A.dbg[blockIdx.x * 16 + 0] = HT_NOW() - t0;
      A.dbg[blockIdx.x * 16 + 1] = w_ae;
      A.dbg[blockIdx.x * 16 + 2] = w_rd;
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================ TMA producer: one box {128 positions, 16 planes} per stage
    if (lane == 0) {
      uint32_t g = 0;
#if CSC_Z_EVICT_FIRST
      const uint64_t zpol = l2_policy_evict_first();
#endif
      for (int j = j0; j < j1; ++j) {
        const int item = h_item_at(A, j);
        const HItem it = h_item(A, item);
        const int plane0 = it.n * A.K + A.ks * A.KC;
        for (int t = 0; t < it.ntiles; ++t) {
          const int pt = it.p0 + 128 * t;  // multiple of 4 floats (BR % 4 == 0): 16-B aligned box start
          for (int c = 0; c < A.NCH; ++c, ++g) {
            const uint32_t slot = g % kHNR, ph = (g / kHNR) & 1u;
            mbar_wait(&rempty[slot], ph ^ 1u);  // the raw tile is free once converted (not once multiplied)
            mbar_arrive_expect_tx(&full[slot], kHRawBytes);
            const uint32_t dst = su32(stg + slot * kHRawBytes);
#if CSC_Z_EVICT_FIRST
            tma_load_2d_hint(dst, &tmap_z, pt, plane0 + 16 * c, &full[slot], zpol);  // {128 positions, 16 planes}
#else
            tma_load_2d(dst, &tmap_z, pt, plane0 + 16 * c, &full[slot]);  // {128 positions, 16 planes}
#endif
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kHEpiBase) {
    // ================================ converters: a pair of warps per stage slot (g mod kHNS = cw / 2)
    // a warp converts whole rows: lane i takes raw floats 4i..4i+3 of row k (one conflict-free 512-B
    // row per warp instruction) and writes their fp16 hi / lo as the 8-B half (i & 1) of the 16-B chunk
    // (i/2) & 7 of atom i/16, swizzled to chunk ((i/2) & 7) ^ (k & 7) (SWIZZLE_128B, MN-major)
    const int cw = warp - kHConvBase;
    const bool want_l1 = A.l1_part != nullptr;
    unsigned long long c_t0 = HT_NOW(), c_wf = 0, c_we = 0;
    const float sz = exp2i(ez);
    double l1 = 0.0;
    uint32_t g = 0;
    const int atom = lane >> 4, cidx = (lane >> 1) & 7, half8 = (lane & 1) * 8;
    // hi = fp16_rn(x_s) (exact in fp16), lo = fp16_rn(x_s - hi) (x_s - hi exact in fp32): packed pair math
    const float2 sz2 = make_float2(sz, sz), mone2 = make_float2(-1.f, -1.f);
    auto split2 = [&](float x0, float x1, uint32_t& hv, uint32_t& lv) {
      const float2 a = __fmul2_rn(make_float2(x0, x1), sz2);
      const __half2 h = __float22half2_rn(a);
      const float2 l = __ffma2_rn(__half22float2(h), mone2, a);
      const __half2 lh = __float22half2_rn(l);
      hv = *reinterpret_cast<const uint32_t*>(&h);
      lv = *reinterpret_cast<const uint32_t*>(&lh);
    };
    (void)split2;
    for (int j = j0; j < j1; ++j) {
      const int item = h_item_at(A, j);
      const HItem it = h_item(A, item);
      for (int t = 0; t < it.ntiles; ++t) {
        const int pt = it.p0 + 128 * t;
        const bool tile_full = pt + 128 <= it.pend;
        for (int c = 0; c < A.NCH; ++c, ++g) {
          if (static_cast<int>(g % kHNS) != (cw >> 1)) continue;
          const uint32_t slot = g % kHNS, ph = (g / kHNS) & 1u;      // hi / lo slot
          const uint32_t rslot = g % kHNR, rph = (g / kHNR) & 1u;  // raw slot
          unsigned long long tw = HT_NOW();
          mbar_wait(&full[rslot], rph);
          unsigned long long tw2 = HT_NOW();
          mbar_wait(&empty[slot], ph ^ 1u);  // the MMA has finished with this slot's previous hi / lo
          c_wf += tw2 - tw;
          c_we += HT_NOW() - tw2;
          const uint8_t* rawp = stg + rslot * kHRawBytes;
          uint8_t* hip = hls + slot * (2 * kHHalfBytes);
          uint8_t* lop = hip + kHHalfBytes;
          float s1 = 0.f;
#pragma unroll 4
          for (int rr = 0; rr < 8; ++rr) {
            const int k = 2 * rr + (cw & 1);  // the pair splits the stage's 16 rows
            const float4 x0 = reinterpret_cast<const float4*>(rawp + k * 512)[lane];
            const int off = atom * 2048 + k * 128 + ((cidx ^ (k & 7)) << 4) + half8;
#if CSC_CH_SPLIT_CVT
            uint2 hv, lv;
            split2(x0.x, x0.y, hv.x, lv.x);
            split2(x0.z, x0.w, hv.y, lv.y);
            *reinterpret_cast<uint2*>(hip + off) = hv;
            *reinterpret_cast<uint2*>(lop + off) = lv;
#else
            const float a0 = x0.x * sz, a1 = x0.y * sz, a2 = x0.z * sz, a3 = x0.w * sz;
            const float h0 = rn11(a0), h1 = rn11(a1), h2 = rn11(a2), h3 = rn11(a3);
            *reinterpret_cast<uint2*>(hip + off) = make_uint2(pack_h2(h0, h1), pack_h2(h2, h3));
            *reinterpret_cast<uint2*>(lop + off) = make_uint2(pack_h2(a0 - h0, a1 - h1), pack_h2(a2 - h2, a3 - h3));
#endif
            if (want_l1) {
              const int kk = A.ks * A.KC + 16 * c + k;  // warp-uniform: padded filter rows add nothing
              if (kk < A.K) {
                if (tile_full) {  // every position of the tile is in the item: no per-value test
                  s1 += (fabsf(x0.x) + fabsf(x0.y)) + (fabsf(x0.z) + fabsf(x0.w));
                } else {
                  const int p = pt + 4 * lane;
                  s1 += (p < it.pend ? fabsf(x0.x) : 0.f) + (p + 1 < it.pend ? fabsf(x0.y) : 0.f) +
                        (p + 2 < it.pend ? fabsf(x0.z) : 0.f) + (p + 3 < it.pend ? fabsf(x0.w) : 0.f);
                }
              }
            }
          }
          if (want_l1) l1 += static_cast<double>(s1);
          fence_async_shared();  // hi / lo writes before the MMA's reads; raw reads before the TMA refill
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&ready[slot]);
            mbar_arrive(&rempty[rslot]);
          }
        }
      }
    }
    const double tsum = warp_sum_d(l1);
    if (lane == 0) l1_warp[cw] = tsum;
    if (A.dbg && cw == 0 && lane == 0) {
      A.dbg[blockIdx.x * 16 + 3] = HT_NOW() - c_t0;
      A.dbg[blockIdx.x * 16 + 4] = c_wf;
      A.dbg[blockIdx.x * 16 + 5] = c_we;
    }
  } else {
    // ================================ epilogue: col2im into one band window (as csc_conv_ss.cu)
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int h = (warp - kHEpiBase) >> 2;  // group of tap rows
    constexpr int AH = (S + kHEpiGroups - 1) / kHEpiGroups;
    const int a_beg = h * AH;
    const int na = min(AH, S - a_beg);      // may be <= 0 for small S
    const float inv = exp2i(-(ez + ef));
    // Wc >= 128 keeps the quarters' window rows disjoint (one pass); narrower rows add in a fixed
    // order of phases (quarters; and their row groups when Wc < 32 + P): deterministic sums
    const int nph = A.Wc >= 128 ? 1 : (A.Wc >= 32 + P ? 4 : 4 * kHEpiGroups);
    const int myph = nph == 1 ? 0 : (nph == 4 ? q : kHEpiGroups * q + h);
    uint32_t tcount = 0;
    unsigned long long e_t0 = HT_NOW(), e_wa = 0, e_red = 0, e_win = 0, e_fl = 0;
    for (int j = j0; j < j1; ++j) {
      const int item = h_item_at(A, j);
      const HItem it = h_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        unsigned long long te = HT_NOW();
        mbar_wait_sleep(&acc_full[buf], use & 1u);
        e_wa += HT_NOW() - te;
        tc_after();
        const int pq = 128 * t + 32 * q;
        const bool pvalid = it.p0 + pq + lane < it.pend;
        const uint32_t tacc = tbase + buf * (A.precise ? 256u : 128u) + (static_cast<uint32_t>(32 * q) << 16);
        float* rowb = win + pq + lane + a_beg * A.Wc;
        float own[AH], dnv[AH];
        // positions past the item's end only occur in its last tile: the common full tile runs
        // without the per-value select
        auto reduce_rows = [&](auto partial) {
          constexpr bool PART = decltype(partial)::value;
#pragma unroll
          for (int i = 0; i < AH; ++i) {
            own[i] = 0.f;
            dnv[i] = 0.f;
            if (i >= na) continue;
            const int a = a_beg + i;
            float y[S];
            tmem_ld_row<S>(tacc + a * S, y);
            if (A.precise) {
              float y2[S];
              tmem_ld_row<S>(tacc + 128u + a * S, y2);
              tmem_ld_wait();
#pragma unroll
              for (int b = 0; b < S; ++b) y[b] += y2[b];
            } else {
              tmem_ld_wait();
            }
            float u0s = 0.f, u1s = 0.f, d0s = 0.f, d1s = 0.f;
#pragma unroll
            for (int b = 0; b < S; ++b) {
              // one rotation serves both parts: lanes >= b get position lane-b of this quarter, lanes < b
              // get position lane-b+32, the halo that belongs to the next quarter's first lanes
              const float yv = PART ? (pvalid ? y[b] : 0.f) : y[b];
              const float rot = b == 0 ? yv : __shfl_sync(kFullMask, yv, (lane - b) & 31);
              if (lane >= b) {
                if (b & 1) u1s += rot; else u0s += rot;
              } else {
                if (b & 1) d1s += rot; else d0s += rot;
              }
            }
            own[i] = u0s + u1s;
            dnv[i] = d0s + d1s;
          }
        };
        const unsigned long long tr0 = HT_NOW();
        if (__all_sync(kFullMask, pvalid)) reduce_rows(std::false_type{});
        else reduce_rows(std::true_type{});
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        const unsigned long long tr1 = HT_NOW();
        e_red += tr1 - tr0;
        if (nph == 1) {
#pragma unroll
          for (int i = 0; i < AH; ++i)
            if (i < na) rowb[i * A.Wc] += own[i];
          named_sync(1, 32 * kHEpiWarps);
          if (lane < P) {
#pragma unroll
            for (int i = 0; i < AH; ++i)
              if (i < na) rowb[i * A.Wc + 32] += dnv[i];
          }
          named_sync(1, 32 * kHEpiWarps);
        } else {
          for (int ph = 0; ph < nph; ++ph) {
            if (ph == myph) {
#pragma unroll
              for (int i = 0; i < AH; ++i)
                if (i < na) rowb[i * A.Wc] += own[i];
              __syncwarp();
              if (lane < P) {
#pragma unroll
                for (int i = 0; i < AH; ++i)
                  if (i < na) rowb[i * A.Wc + 32] += dnv[i];
              }
            }
            named_sync(1, 32 * kHEpiWarps);
          }
        }
        e_win += HT_NOW() - tr1;
      }
      const unsigned long long tf0 = HT_NOW();
      float* dst = A.part + (static_cast<size_t>(it.n) * A.nbands + (it.u0 / A.BR)) *
                                static_cast<size_t>(A.BR + P) * A.W;
      const int rows = A.BR + P;
      const int et = tid - 32 * kHEpiBase;
      for (int e = et; e < rows * A.W; e += 32 * kHEpiWarps) {
        const int r = e / A.W, j = e - r * A.W;
        const float v = win[r * A.Wc + j + P] * inv;  // exact: power of two
        dst[e] = A.ks == 0 ? v : dst[e] + v;
      }
      named_sync(1, 32 * kHEpiWarps);
      for (int e = et; e < A.WL; e += 32 * kHEpiWarps) win[e] = 0.f;
      named_sync(1, 32 * kHEpiWarps);
      e_fl += HT_NOW() - tf0;
    }
    if (A.dbg && warp == kHEpiBase && lane == 0) {
      A.dbg[blockIdx.x * 16 + 6] = HT_NOW() - e_t0;
      A.dbg[blockIdx.x * 16 + 7] = e_wa;
      A.dbg[blockIdx.x * 16 + 8] = e_red;
      A.dbg[blockIdx.x * 16 + 9] = e_win;
      A.dbg[blockIdx.x * 16 + 10] = e_fl;
    }
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
  if (tid == 0 && A.l1_part != nullptr) {
    double s = 0.0;
    for (int i = 0; i < kHConvWarps; ++i) s += l1_warp[i];
    A.l1_part[static_cast<size_t>(A.ks) * gridDim.x + blockIdx.x] = s;
  }
}

// B image (16 blocks, each computing the same max |f| -> fmax, float bits); then, with 2^ef, the fp16 hi/lo image
// bimg[ks][hl][atom][k][64 taps] in the MN-major SW128 layout (16-B chunk (t%64)/8 XOR (k%8)).
__global__ void __launch_bounds__(1024) bimg_h_kernel(const float* __restrict__ f, int K, int S2, int KC, int nks,
                                                      uint16_t* __restrict__ bimg, uint32_t* __restrict__ fmax) {
  __shared__ uint32_t mx;
  if (threadIdx.x == 0) mx = 0u;
  __syncthreads();
  uint32_t m = 0u;
  // 8 independent loads in flight per thread (the max over K*S2 values is latency-bound)
  const int nf = K * S2;
  for (int e0 = threadIdx.x; e0 < nf; e0 += 8 * blockDim.x) {
    float fv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      fv[u] = e < nf ? __ldg(f + e) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) m = max(m, __float_as_uint(fabsf(fv[u])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFullMask, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&mx, m);
  __syncthreads();
  const uint32_t mbits = mx;
  if (threadIdx.x == 0 && blockIdx.x == 0) *fmax = mbits;
  const float sf = exp2i(scale_exp(mbits));
  const int total = nks * KC * 128;
  // every block finds the (same) max over the small filter tensor, then writes its share
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int t = e & 127;
    const int k = (e >> 7) % KC, ks = (e >> 7) / KC;
    const int kg = ks * KC + k;
    const float v = (kg < K && t < S2) ? f[static_cast<size_t>(kg) * S2 + t] * sf : 0.f;
    const float hv = rn11(v);
    const __half hh = __float2half_rn(hv), hl = __float2half_rn(v - hv);
    const int atom = t >> 6, tt = t & 63;
    const size_t blk = static_cast<size_t>(2) * KC * 64;  // halves per (ks, hl)
    const size_t off = static_cast<size_t>(atom) * KC * 64 + static_cast<size_t>(k) * 64 +
                       ((((tt >> 3) ^ (k & 7))) << 3) + (tt & 7);
    bimg[(static_cast<size_t>(ks) * 2 + 0) * blk + off] = *reinterpret_cast<const uint16_t*>(&hh);
    bimg[(static_cast<size_t>(ks) * 2 + 1) * blk + off] = *reinterpret_cast<const uint16_t*>(&hl);
  }
}

// max |x| as the bits of a non-negative float (monotone in the value).  float4 loads when x is
// 16-B aligned; a block-level reduction and one global atomic per block (per-warp atomics on one
// address serialise at L2: 4.7k of them cost 40 us).
__global__ void absmax_kernel(const float* __restrict__ x, int64_t n, int vec, uint32_t* __restrict__ out) {
  __shared__ uint32_t red;
  if (threadIdx.x == 0) red = 0u;
  __syncthreads();
  uint32_t m = 0u;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t tail = 0;
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t n4 = n / 4;
    for (int64_t i = t0; i < n4; i += stride) {
      const float4 v = __ldg(x4 + i);
      m = max(max(m, __float_as_uint(fabsf(v.x))), max(__float_as_uint(fabsf(v.y)), __float_as_uint(fabsf(v.z))));
      m = max(m, __float_as_uint(fabsf(v.w)));
    }
    tail = n4 * 4;
  }
  for (int64_t i = tail + t0; i < n; i += stride) m = max(m, __float_as_uint(fabsf(x[i])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFullMask, m, o));
  if ((threadIdx.x & 31) == 0 && m != 0u) atomicMax(&red, m);
  __syncthreads();
  if (threadIdx.x == 0 && red != 0u) atomicMax(out, red);
}

template <int S>
cudaError_t run_conv_h(const CUtensorMap& tm, const HArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&conv_h_kernel<S>), kHSmemMax);
  if (e != cudaSuccess) return e;
#ifdef CSC_ROLE_TIMING
  static unsigned long long* dbg = nullptr;
  static int calls = 0;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 16 * 1024);
  cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 16 * 1024, st);
  HArgs b = a;
  b.dbg = dbg;
  conv_h_kernel<S><<<grid, kHThreads, smem, st>>>(tm, b);
  if (++calls % 4 == 0) {
    static unsigned long long h[16 * 1024];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost);
    double t[16] = {0};
    for (int bk = 0; bk < grid; ++bk)
      for (int i = 0; i < 16; ++i) t[i] += static_cast<double>(h[bk * 16 + i]) / grid;
    fprintf(stderr,
            "[conv_h roles p%d] mma: total %.0f w_accempty %.0f w_ready %.0f | conv0: total %.0f w_full %.0f w_empty %.0f | "
            "epi0: total %.0f w_accfull %.0f reduce %.0f window %.0f flush %.0f\n",
            a.precise, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], t[9], t[10]);
  }
#else
  conv_h_kernel<S><<<grid, kHThreads, smem, st>>>(tm, a);
#endif
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- host side
bool conv_h_supported(const Geom& g) {
  return (g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) && g.N > 0 &&
         (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 && tc_ntaps_padded(g.S) <= 128 && tmap_available();
}

// Longest-processing-time-first assignment of the items (image, band of BR code rows; cost = its 128-position
// tiles + overhead for the band's staging / window flush) to the G persistent CTAs: each item in decreasing cost goes to the
// least-loaded CTA (ties: lowest index).  Writes [G + 1] CTA offsets, then the items CTA by CTA (in the order
// assigned), and returns the largest CTA load in tiles.  Round robin (item = CTA + j * G) leaves the CTA
// with one item more than the others idle-free while the rest wait: at config 3 with BR = 8 the busiest CTA
// had 170 tiles against a mean of 153.
int64_t lpt_bands(const Geom& g, int BR, int G, int overhead, std::vector<int>* out) {
  const int nb = ceil_div(g.Hc, BR);
  const int nitems = g.N * nb;
  std::vector<int64_t> cost(nb);
  for (int b = 0; b < nb; ++b) {
    const int u0 = b * BR, u1 = std::min(u0 + BR, g.Hc);
    cost[b] = ceil_div((u1 - u0) * g.Wc, 128) + overhead;
  }
  // stable order of decreasing cost (items of one cost keep their image-major order)
  std::vector<int> order(nitems);
  for (int i = 0; i < nitems; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a % nb] > cost[b % nb]; });
  using E = std::pair<int64_t, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
  for (int c = 0; c < G; ++c) pq.push(E(0, c));
  std::vector<std::vector<int>> per(out ? G : 0);
  int64_t mx = 0;
  for (int i : order) {
    E e = pq.top();
    pq.pop();
    e.first += cost[i % nb];
    mx = std::max(mx, e.first);
    if (out) per[e.second].push_back(i);
    pq.push(e);
  }
  if (out) {
    out->assign(G + 1 + nitems, 0);
    int j = 0;
    for (int c = 0; c < G; ++c) {
      (*out)[c] = j;
      for (int i : per[c]) (*out)[G + 1 + j++] = i;
    }
    (*out)[G] = j;
  }
  return mx;
}

bool conv_h_plan(const Geom& g, int num_sms, TcPlan& p) {
  p = TcPlan{};
  p.NT = 128;  // taps padded to 2 atoms of 64
  p.natoms = 2;
  const int stages = kHRingBytes;
  auto wl = [&](int br) { return (br + g.P) * g.Wc + 192; };
  int kc_fit = (kHSmemMax - 2048 - stages - wl(4) * 4) / (2 * 2 * 128);
  kc_fit = kc_fit / 16 * 16;
  if (kc_fit > 128) kc_fit = 128;
  if (kc_fit < 16) return false;
  p.nks = ceil_div(g.K, kc_fit);
  p.KC = (ceil_div(g.K, p.nks) + 15) / 16 * 16;
  p.NCH = p.KC / 16;
  const int bsm = 2 * 2 * p.KC * 128;
  // band height: every BR that fits (BR * Wc % 4 == 0: 16-B aligned TMA box starts), the smallest busiest-CTA
  // load under the LPT schedule; on ties the taller band (fewer halo rows in the partials the fixup reads)
  const int G = std::max(1, std::min(num_sms, g.N * ceil_div(g.Hc, 4)));
  int BR = 0;
  int64_t best = 0;
  for (int br = 1; br <= 32 && br <= std::max(g.Hc, 4); ++br) {
    if ((static_cast<int64_t>(br) * g.Wc) % 4 != 0) continue;
    if (2048 + bsm + stages + wl(br) * 4 > kHSmemMax) break;
    if (g.N <= 0) {
      BR = br;
      continue;
    }
    const int64_t c = lpt_bands(g, br, std::min(G, g.N * ceil_div(g.Hc, br)), 1, nullptr);
    if (BR == 0 || c <= best) {
      BR = br;
      best = c;
    }
  }
  if (BR == 0) return false;
  p.BR = BR;
  p.WL = wl(BR);
  p.nbands = ceil_div(g.Hc, BR);
  p.nitems = g.N * p.nbands;
  p.grid = p.nitems < num_sms ? p.nitems : num_sms;
  if (p.grid < 1) p.grid = 1;
  p.smem = 1024 + bsm + stages + p.WL * 4;
  p.part_floats = static_cast<size_t>(g.N) * p.nbands * (p.BR + g.P) * g.W;
  p.bimg_floats = static_cast<size_t>(p.nks) * 2 * 2 * p.KC * 64 / 2 + 16;  // fp16 image, in floats
  p.ss = false;
  p.half = true;
  return true;
}

void conv_h_schedule(const Geom& g, const TcPlan& p, std::vector<int>& out) {
  if (g.N <= 0 || p.nitems <= 0) {
    out.assign(p.grid + 1, 0);
    return;
  }
  lpt_bands(g, p.BR, p.grid, 1, &out);
}

cudaError_t launch_absmax(const float* x, int64_t n, uint32_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  const int vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 ? 1 : 0;
  if (n > 0) absmax_kernel<<<148 * 4, 256, 0, st>>>(x, n, vec, out);
  return cudaGetLastError();
}

cudaError_t launch_conv_h(const Geom& g, const TcPlan& p, TmapCache* tmc, const float* z, const float* filt,
                          float* bimg_f, const uint32_t* zmax, uint32_t* fmax, float* part, double* l1_part,
                          cudaStream_t st, bool build_b, bool precise) {
  const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
  cudaError_t e0 = tmap_2d(*tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K, plane * 4,
                           128, 16, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (e0 != cudaSuccess) return e0;
  const CUtensorMap& tm = tmc->map;
  uint16_t* bimg = reinterpret_cast<uint16_t*>(bimg_f);
  if (build_b) bimg_h_kernel<<<16, 1024, 0, st>>>(filt, g.K, g.S * g.S, p.KC, p.nks, bimg, fmax);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  HArgs a{};
  a.bimg = bimg;
  a.zmax = zmax;
  a.fmax = fmax;
  a.part = part;
  a.l1_part = l1_part;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.NCH = p.NCH; a.NT = p.NT;
  a.BR = p.BR; a.nbands = p.nbands; a.nitems = p.nitems; a.WL = p.WL;
  a.precise = precise ? 1 : 0;
  a.sched = p.sched;
  for (int ks = 0; ks < p.nks; ++ks) {
    a.ks = ks;
    switch (g.S) {
      case 5: e = run_conv_h<5>(tm, a, p.grid, p.smem, st); break;
      case 7: e = run_conv_h<7>(tm, a, p.grid, p.smem, st); break;
      case 9: e = run_conv_h<9>(tm, a, p.grid, p.smem, st); break;
      case 11: e = run_conv_h<11>(tm, a, p.grid, p.smem, st); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace csc

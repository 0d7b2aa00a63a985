// csc_wgrad_h.cu -- filter gradient g = Z^T r' on the sm_100a tensor cores at the fp16 rate
// (tcgen05.mma kind::f16, 3-term split, fp32 accumulate), TMA-fed.
//
// Gradient of the Eq.5 fit term (§3.1): for every filter k and tap t = (a, b)
//   g[k][t] = sum_n sum_{(u,v)} z[n,k,u,v] * R_n[(u,v)][t],   R_n[(u,v)][(a,b)] = r'[n, u-P+a, v-P+b]
// (r' = 0 outside the H x W image).  As a GEMM per CTA:  D[t][k] += sum_pos A[t][pos] B[k][pos],
//   M = 128 taps (s^2 <= 121 used), N = Npad filters of one k-group, K = code positions, 16 per MMA.
// Both operands are split after exact power-of-two scalings (reading T6, as csc_conv_h.cu):
//   x_s = x 2^e,  hi = fp16_rn(x_s) (z) or rn11(x_s) (r'),  lo = fp16_rn(x_s - hi)  (x_s - hi is exact in fp32),
//   D += A_hi B_hi + A_hi B_lo + A_lo B_hi   (2^-22 per product, like 3xTF32, at twice its rate).
// e_z from the running bound of max|z| (the code step raises it), e_r from max|r'|.
// Operands:
//   B = z: one TMA box {64 positions, KC planes} (fp32) per chunk into a ring of raw slots (one request per
//       chunk: the producer's issue rate stays off the critical path); the converter warps write the scaled
//       fp16 hi / lo rows in the canonical K-major SWIZZLE_128B layout (row = filter, 128 B = 64 positions,
//       16-B chunks XOR row) and release the raw slot at once.
//   A = im2col of r' in TMEM (lane = tap, one 32-bit column = two consecutive positions): the item's
//       residual rows are staged by cp.async and split into fp16 PAIRS (double-buffered, one item ahead, by the
//       otherwise idle epilogue warps) hp[row][c] =
//       (hi(r[c]), hi(r[c+1])), so a column is one shared load per lane (pitch = s mod 32: the 32 taps of
//       a lane quarter hit 32 banks).
// The accumulator restarts every tile (cpt chunks); the epilogue adds it into fp32 block sums that are
// flushed into the CTA's fp64 partials every 2048 positions, and wgrad_reduce_kernel sums the per-CTA
// partials in a fixed order (deterministic), exactly as csc_wgrad_tc.cu.
//
// CTA (persistent, 32 warps): warp 0 MMA, warp 1 TMA, warps 2..7 z converters (all of them on every chunk),
// warps 8..15 im2col (two groups of 4 lane quarters, alternate chunks), warps 16..31 epilogue (4 per quarter).
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
#include <cuda_runtime.h>

#ifndef CSC_Z_EVICT_FIRST
#define CSC_Z_EVICT_FIRST 1  // stream z through L2 evict-first (tcx::tma_load_2d_hint): 0.390 -> 0.378 ms
#endif

namespace csc {
namespace {

using namespace tcx;

constexpr int kWhNRMax = 8;      // raw TMA slots (one {64 positions, KC planes} box = one chunk each)
constexpr int kWhNA = 4;         // TMEM A slots (64 columns each: 4 K16-steps x (8 hi + 8 lo))
constexpr int kWhZWarps = 10;
constexpr int kWhIGroups = 1;    // groups of 4 lane-quarter warps; group g takes the chunks c with c % groups == g
constexpr int kWhIWarps = 4 * kWhIGroups;
constexpr int kWhEpiWarps = 16;
constexpr int kWhZBase = 2, kWhIBase = kWhZBase + kWhZWarps, kWhEpiBase = kWhIBase + kWhIWarps;
constexpr int kWhWarps = kWhEpiBase + kWhEpiWarps;
constexpr int kWhThreads = 32 * kWhWarps;
constexpr int kWhChunk = 64;       // positions per chunk (one SW128 atom of fp16 along K)
constexpr int kWhFlushPos = 2048;  // positions summed in fp32 (tensor core + epilogue) before each fp64 flush
constexpr int kWhSmemMax = 226 * 1024;
constexpr uint32_t kWhColA = 256;

__host__ __device__ constexpr uint32_t idesc_f16_kk_w(int M, int N) {  // fp16 A/B K-major, fp32 D
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (0u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ int scale_exp_w(uint32_t mbits) {  // 2^e with m 2^e < 2^14
  if ((mbits & 0x7FFFFFFFu) == 0u) return 0;
  const int E = static_cast<int>((mbits >> 23) & 0xFFu) - 127;
  int e = 13 - E;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}
__device__ __forceinline__ float exp2i_w(int e) { return __uint_as_float(static_cast<uint32_t>(e + 127) << 23); }
__device__ __forceinline__ float rn11_w(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ uint32_t pack_h2_w(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

#ifdef CSC_ROLE_TIMING
#define WT_NOW() clock64()
#define WT_ACC(var, stmt)                       \
  do {                                          \
    const unsigned long long _t = clock64();    \
    stmt;                                       \
    var += clock64() - _t;                      \
  } while (0)
#else
#define WT_NOW() 0ull
#define WT_ACC(var, stmt) stmt
#endif

struct WhArgs {
  const float* r;        // [N][H][W]
  const uint32_t* zmax;  // bound on max|z| (float bits)
  const uint32_t* rmax;  // max|r| (float bits)
  double* gpart;         // [G][K][S*S]
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, NCH, nkg, G;
  int L, nseg, nitems;
  int pitch, rs_rows, rs_floats;
  int NB, NR, cpt;
  unsigned long long* dbg;  // CSC_ROLE_TIMING builds: per-CTA role cycle counters [grid][16]
};

// position in a ring of n slots: slot index and the parity of the pass over the ring (no runtime modulo)
struct Ring {
  uint32_t slot = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++slot == n) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

struct WhItem {
  int n, p0, p1, nch, u_first;
};
__device__ __forceinline__ WhItem wh_item(const WhArgs& A, int item) {
  WhItem it;
  it.n = item / A.nseg;
  const int sg = item - it.n * A.nseg;
  const int plane = A.Hc * A.Wc;
  it.p0 = sg * A.L;
  it.p1 = min(it.p0 + A.L, plane);
  it.nch = (it.p1 - it.p0 + kWhChunk - 1) / kWhChunk;
  it.u_first = it.p0 / A.Wc;
  return it;
}

template <int NC>
__global__ void __launch_bounds__(kWhThreads, 1)
wgrad_h_kernel(const __grid_constant__ CUtensorMap tmap_z, const WhArgs A) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t raw_full[kWhNRMax], raw_empty[kWhNRMax];
  __shared__ __align__(8) uint64_t b_ready[8], b_empty[8], a_ready[kWhNA], a_empty[kWhNA], acc_full[2], acc_empty[2];
  __shared__ __align__(8) uint64_t pair_full[2], pair_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int bbytes = A.Npad * 128;                       // one of hi / lo of a chunk
  uint8_t* bst = sm;                                     // [NB][hi | lo]
  const int rawbytes = A.KC * kWhChunk * 4;             // one TMA box {64 positions, KC planes} fp32
  uint8_t* rawst = bst + 2 * A.NB * bbytes;              // [NR][KC][64] fp32
  // residual pairs, double-buffered per item: [2][hi | lo][rs_rows][pitch]; rstage = raw rows of the next item
  uint32_t* pairs = reinterpret_cast<uint32_t*>(rawst + A.NR * rawbytes);
  float* rstage = reinterpret_cast<float*>(pairs + 4 * A.rs_floats);
  const int ez = scale_exp_w(*A.zmax), er = scale_exp_w(*A.rmax);

  // B rows KC .. Npad-1 (padding filters) stay zero: the converters write rows < KC only
  for (int e = tid; e < 2 * A.NB * bbytes / 16; e += kWhThreads) reinterpret_cast<int4*>(bst)[e] = make_int4(0, 0, 0, 0);
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < A.NR; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], kWhZWarps);
    }
    for (int i = 0; i < A.NB; ++i) {
      mbar_init(&b_ready[i], kWhZWarps);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < kWhNA; ++i) {
      mbar_init(&a_ready[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kWhEpiWarps);
      mbar_init(&pair_full[i], kWhEpiWarps);
      mbar_init(&pair_empty[i], kWhIWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 1 && lane == 0) tma_prefetch_desc(&tmap_z);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  const uint32_t t_acc = tbase;            // 2 x Npad columns
  const uint32_t t_a = tbase + kWhColA;    // kWhNA slots x 64 columns

  if (warp == 0) {
    // ================================ MMA issuer
    const uint32_t idesc = idesc_f16_kk_w(128, A.Npad);
    uint32_t tcount = 0;
    Ring rb, ra;
    unsigned long long t0 = WT_NOW(), w_acc = 0, w_b = 0, w_a = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      const int ntl = (it.nch + A.cpt - 1) / A.cpt;
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        WT_ACC(w_acc, mbar_wait_sleep(&acc_empty[buf], (use & 1u) ^ 1u));
        tc_after();
        const uint32_t d = t_acc + buf * static_cast<uint32_t>(A.Npad);
        const int c0 = tl * A.cpt, c1 = min(c0 + A.cpt, it.nch);
        for (int c = c0; c < c1; ++c, rb.next(A.NB), ra.next(kWhNA)) {
          const uint32_t bs = rb.slot, as = ra.slot;
          WT_ACC(w_b, mbar_wait_sleep(&b_ready[bs], rb.ph));
          WT_ACC(w_a, mbar_wait_sleep(&a_ready[as], ra.ph));
          tc_after();
          const int nks = min(4, (it.p1 - it.p0 - kWhChunk * c + 15) >> 4);
          const uint32_t sh = su32(bst + bs * 2 * bbytes), sl = sh + bbytes;
          const uint32_t ah = t_a + as * 64u;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e < nks) {
              const uint64_t bh = sdesc(sh + 32u * e, 16u, 1024u, kLayout128B);
              const uint64_t bl = sdesc(sl + 32u * e, 16u, 1024u, kLayout128B);
              const uint32_t acc0 = (c > c0 || e > 0) ? 1u : 0u;
              asm volatile(
                  "{\n.reg .pred e, p, t;\n"
                  "elect.sync _|e, 0xffffffff;\n"
                  "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %4, p;\n"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %6, %4, t;\n"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %4, t;\n"
                  "}\n" ::"r"(d),
                  "r"(ah + 8u * e), "r"(ah + 32u + 8u * e), "l"(bh), "r"(idesc), "r"(acc0), "l"(bl)
                  : "memory");
            }
          }
          mma_commit_elect(&b_empty[bs]);
          mma_commit_elect(&a_empty[as]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    if (A.dbg && lane == 0) {
      unsigned long long* o = A.dbg + blockIdx.x * 16;
      o[0] = WT_NOW() - t0; o[1] = w_acc; o[2] = w_b; o[3] = w_a;
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================ TMA producer: one box {64 positions, KC planes} per chunk
    if (lane == 0) {
      Ring rr;
      const int plane0 = kg * A.KC;
#if CSC_Z_EVICT_FIRST
      const uint64_t zpol = l2_policy_evict_first();
#endif
      unsigned long long t0 = WT_NOW(), w_e = 0;
      for (int item = gi; item < A.nitems; item += A.G) {
        const WhItem it = wh_item(A, item);
        for (int c = 0; c < it.nch; ++c, rr.next(A.NR)) {
          const uint32_t slot = rr.slot;
          WT_ACC(w_e, mbar_wait_sleep(&raw_empty[slot], rr.ph ^ 1u));
          mbar_arrive_expect_tx(&raw_full[slot], static_cast<uint32_t>(rawbytes));
          // the inner coordinate p0 + 64 c is a multiple of 4 floats: a 16-B aligned box start (positions
          // past the plane end are zero-filled; those past the item meet zero im2col columns)
#if CSC_Z_EVICT_FIRST
          tma_load_2d_hint(su32(rawst + slot * rawbytes), &tmap_z, it.p0 + kWhChunk * c, it.n * A.K + plane0,
                           &raw_full[slot], zpol);
#else
          tma_load_2d(su32(rawst + slot * rawbytes), &tmap_z, it.p0 + kWhChunk * c, it.n * A.K + plane0,
                      &raw_full[slot]);
#endif
        }
      }
      if (A.dbg) {
        unsigned long long* o = A.dbg + blockIdx.x * 16;
        o[4] = WT_NOW() - t0; o[5] = w_e;
      }
    }
    __syncwarp();
  } else if (warp < kWhIBase) {
    // ================================ z converters: every warp converts row pairs w, w + 6, ... of every chunk.
    // lane i, row pair rp: row k = 2 rp + i / 16, positions 4 (i % 16) .. +3 (one float4: a 512-B warp read),
    // written as the 8-B half (i & 1) of the 16-B chunk (i % 16) / 2 of row k, swizzled to ((i % 16) / 2) ^ (k & 7)
    const int zw = warp - kWhZBase;
    const float sz = exp2i_w(ez);
    const float2 sz2 = make_float2(sz, sz), mone2 = make_float2(-1.f, -1.f);
    const int cidx = (lane & 15) >> 1, half8 = (lane & 1) * 8;
    const int npairs = (A.KC + 1) >> 1;
    Ring rr, rb;
    unsigned long long t0 = WT_NOW(), w_f = 0, w_be = 0;
    // hi = fp16_rn(x_s) (exact in fp16), lo = fp16_rn(x_s - hi) (x_s - hi exact in fp32): packed pair math
    auto split2 = [&](float x0, float x1, uint32_t& hv, uint32_t& lv) {
      const float2 a = __fmul2_rn(make_float2(x0, x1), sz2);
      const __half2 h = __float22half2_rn(a);
      const float2 l = __ffma2_rn(__half22float2(h), mone2, a);
      const __half2 lh = __float22half2_rn(l);
      hv = *reinterpret_cast<const uint32_t*>(&h);
      lv = *reinterpret_cast<const uint32_t*>(&lh);
    };
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      for (int c = 0; c < it.nch; ++c, rr.next(A.NR), rb.next(A.NB)) {
        const uint32_t slot = rr.slot, bs = rb.slot;
        WT_ACC(w_f, mbar_wait_sleep(&raw_full[slot], rr.ph));
        WT_ACC(w_be, mbar_wait_sleep(&b_empty[bs], rb.ph ^ 1u));  // the MMA is done with the stage's previous chunk
        const uint8_t* rp = rawst + slot * rawbytes + (lane & 15) * 16;
        uint8_t* hip = bst + bs * 2 * bbytes + half8;
        uint8_t* lop = hip + bbytes;
#pragma unroll 3
        for (int pr = zw; pr < npairs; pr += kWhZWarps) {
          const int k = 2 * pr + (lane >> 4);
          if (k < A.KC) {
            const float4 x = *reinterpret_cast<const float4*>(rp + k * 256);
            uint2 hv, lv;
            split2(x.x, x.y, hv.x, lv.x);
            split2(x.z, x.w, hv.y, lv.y);
            const int off = k * 128 + ((cidx ^ (k & 7)) << 4);
            *reinterpret_cast<uint2*>(hip + off) = hv;
            *reinterpret_cast<uint2*>(lop + off) = lv;
          }
        }
        fence_async_shared();  // generic writes before the MMA's async-proxy reads; raw reads before the refill
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&raw_empty[slot]);
          mbar_arrive(&b_ready[bs]);
        }
      }
    }
    if (A.dbg && zw == 0 && lane == 0) {
      unsigned long long* o = A.dbg + blockIdx.x * 16;
      o[6] = WT_NOW() - t0; o[7] = w_f; o[8] = w_be;
    }
  } else if (warp < kWhEpiBase) {
    // ================================ im2col: lane = tap t = 32 q + lane, two positions per TMEM column;
    // group grp of 4 warps takes the chunks of its parity (two chunks in flight)
    const int iw = warp - kWhIBase;
    const int q = iw & 3, grp = iw >> 2;
    const int it_tid = tid - 32 * kWhIBase;  // 0..255
    const int t = 32 * q + lane;
    const int S2 = A.S * A.S;
    const int ta = t < S2 ? t / A.S : 0, tb = t < S2 ? t - ta * A.S : 0;
    const int toff = ta * A.pitch + tb;  // taps past s^2 read offset 0 (finite; their D rows are never read)
    const uint32_t tq = static_cast<uint32_t>(32 * q) << 16;
    uint32_t cc = 0, ii = 0;
    unsigned long long t0 = WT_NOW(), w_ae = 0, w_fill = 0;
    for (int item = gi; item < A.nitems; item += A.G, ++ii) {
      const WhItem it = wh_item(A, item);
      const uint32_t pb = ii & 1u;
      WT_ACC(w_fill, mbar_wait_sleep(&pair_full[pb], (ii >> 1) & 1u));  // the epilogue warps built this item's pairs
      const uint32_t* hp = pairs + pb * 2 * A.rs_floats;
      const uint32_t* lp = hp + A.rs_floats;
      const uint32_t* sh = hp + toff;
      const uint32_t* sl = lp + toff;
      for (int c = 0; c < it.nch; ++c, ++cc) {
        if (kWhIGroups > 1 && static_cast<int>(cc % kWhIGroups) != grp) continue;
        const uint32_t as = cc % kWhNA;
        WT_ACC(w_ae, mbar_wait_sleep(&a_empty[as], ((cc / kWhNA) & 1u) ^ 1u));
        tc_after();
        const int pk = it.p0 + kWhChunk * c;
        int u = pk / A.Wc;
        int v = pk - u * A.Wc;
        const uint32_t col0 = t_a + as * 64u;
        if (v + kWhChunk <= A.Wc && pk + kWhChunk <= it.p1) {
          // the chunk lies in one code row: 32 aligned pairs of one residual row
          const int o = (u - it.u_first) * A.pitch + v;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              hv[jj] = sh[o + 16 * e + 2 * jj];
              lv[jj] = sl[o + 16 * e + 2 * jj];
            }
            tmem_st8(tq + col0 + 8u * e, hv);
            tmem_st8(tq + col0 + 32u + 8u * e, lv);
          }
        } else if ((A.Wc & 1) == 0 && A.Wc >= kWhChunk && pk + kWhChunk <= it.p1) {
          // the chunk wraps into the next code row (once: Wc >= 64); Wc even: positions start even, so no pair
          // straddles two rows
          const int o0 = (u - it.u_first) * A.pitch;
          const int o1 = o0 + A.pitch - A.Wc;  // offset of position v' >= Wc (row u + 1, column v' - Wc)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int vv = v + 16 * e + 2 * jj;
              const int o = (vv < A.Wc ? o0 : o1) + vv;
              hv[jj] = sh[o];
              lv[jj] = sl[o];
            }
            tmem_st8(tq + col0 + 8u * e, hv);
            tmem_st8(tq + col0 + 32u + 8u * e, lv);
          }
        } else {
          // row wraps (a pair may straddle two rows when Wc is odd) or the end of the item
#pragma unroll 1
          for (int e = 0; e < 4; ++e) {
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int pp = pk + 16 * e + 2 * jj;
              uint32_t xh = 0u, xl = 0u;
              if (pp < it.p1) {
                const int o0 = (u - it.u_first) * A.pitch + v;
                if (v + 1 < A.Wc) {
                  xh = sh[o0];
                  xl = sl[o0];
                  if (pp + 1 >= it.p1) {
                    xh &= 0xFFFFu;
                    xl &= 0xFFFFu;
                  }
                } else {
                  const int o1 = (u + 1 - it.u_first) * A.pitch;
                  const bool two = pp + 1 < it.p1;
                  xh = __byte_perm(sh[o0], two ? sh[o1] : 0u, 0x5410);
                  xl = __byte_perm(sl[o0], two ? sl[o1] : 0u, 0x5410);
                }
              }
              hv[jj] = xh;
              lv[jj] = xl;
              v += 2;
              if (v >= A.Wc) {
                v -= A.Wc;
                ++u;
              }
            }
            tmem_st8(tq + col0 + 8u * e, hv);
            tmem_st8(tq + col0 + 32u + 8u * e, lv);
          }
        }
        tmem_st_wait();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_ready[as]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pair_empty[pb]);  // done reading this item's pairs
    }
    if (A.dbg && iw == 0 && lane == 0) {
      unsigned long long* o = A.dbg + blockIdx.x * 16;
      o[9] = WT_NOW() - t0; o[10] = w_ae; o[11] = w_fill;
    }
  } else {
    // ================================ epilogue: D[t][k] (fp32, per tile) -> fp32 block sums -> fp64 partials
    const int ew = warp - kWhEpiBase;  // 0..15
    const int q = warp & 3;
    const int cb = ew >> 2;            // column block (NC columns)
    const int t = 32 * q + lane;
    const int S2 = A.S * A.S;
    const float inv = exp2i_w(-(ez + er));
    float acc[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = 0.f;
    int nacc = 0;
    bool first = true;
    double* const gp0 = A.gpart + (static_cast<size_t>(gi) * A.K + kg * A.KC + cb * NC) * S2 + t;
    const int nvalid = min(NC, min(A.KC - cb * NC, A.K - kg * A.KC - cb * NC));
    auto flush = [&]() {
      if (t < S2) {
        // the first block is stored, later ones are added with fire-and-forget fp64 reductions; one thread
        // owns each element and same-address operations of a thread keep program order: deterministic
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          if (i < nvalid) {
            double* gp = gp0 + static_cast<size_t>(i) * S2;
            const double v = static_cast<double>(acc[i] * inv);  // exact: a power of two
            if (first) *gp = v;
            else atomicAdd(gp, v);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) acc[i] = 0.f;
      first = false;
      nacc = 0;
    };
    const uint32_t tq = static_cast<uint32_t>(32 * q) << 16;
    const int flush_tiles = max(1, kWhFlushPos / (kWhChunk * A.cpt));
    // The epilogue warps (idle most of the time) also build the im2col's residual pairs, one item ahead:
    // rstage[rho][c] = r'[n, u_first - P + rho, c - P] (0 outside the image) by cp.async one fill ahead, then
    // scaled and split into hp[rho][c] = (hi(t[c]), hi(t[c+1])), lp likewise, in pair buffer (item & 1)
    const int et = tid - 32 * kWhEpiBase;  // 0..511
    const float sr = exp2i_w(er);
    auto stage = [&](int item) {
      const WhItem it = wh_item(A, item);
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      const int st_dc = (32 * kWhEpiWarps) % A.pitch, st_dr = (32 * kWhEpiWarps) / A.pitch;
      const uint32_t st_dst0 = su32(rstage);
      int c = et % A.pitch, rho = et / A.pitch;  // this thread's first element (row, column)
      for (int e = et; e < A.rs_floats; e += 32 * kWhEpiWarps) {
        const int i = it.u_first - A.P + rho, jc = c - A.P;
        const bool ok = i >= 0 && i < A.H && jc >= 0 && jc < A.W;
        cp_async4(st_dst0 + 4u * static_cast<uint32_t>(e), ok ? rn + static_cast<size_t>(i) * A.W + jc : rn, ok);
        c += st_dc;
        rho += st_dr;
        if (c >= A.pitch) {
          c -= A.pitch;
          ++rho;
        }
      }
      cp_async_commit();
    };
    // pairs of the ii-th item of this CTA (its rows are staged); then stage the rows of the next one
    auto fill = [&](uint32_t ii, int item) {
      const uint32_t pb = ii & 1u;
      mbar_wait_sleep(&pair_empty[pb], ((ii >> 1) & 1u) ^ 1u);  // the im2col is done with item ii - 2
      cp_async_wait<0>();
      named_sync(2, 32 * kWhEpiWarps);
      uint32_t* hp = pairs + pb * 2 * A.rs_floats;
      uint32_t* lp = hp + A.rs_floats;
      for (int e = et; e < A.rs_floats; e += 32 * kWhEpiWarps) {
        const float x0 = rstage[e] * sr;
        const float x1 = (e + 1 < A.rs_floats ? rstage[e + 1] : 0.f) * sr;
        const float h0 = rn11_w(x0), h1 = rn11_w(x1);
        hp[e] = pack_h2_w(h0, h1);
        lp[e] = pack_h2_w(x0 - h0, x1 - h1);
      }
      named_sync(2, 32 * kWhEpiWarps);  // every epilogue thread is done reading rstage
      if (item + A.G < A.nitems) stage(item + A.G);
      __syncwarp();
      if (lane == 0) mbar_arrive(&pair_full[pb]);
    };
    if (gi < A.nitems) {
      stage(gi);
      fill(0u, gi);
    }
    uint32_t ii = 0;
    constexpr int NB4 = 2;  // x4 loads per batch (the 64-register cap at 1024 threads)
    uint32_t tcount = 0;
    unsigned long long t0 = WT_NOW(), w_af = 0;
    for (int item = gi; item < A.nitems; item += A.G, ++ii) {
      const WhItem it = wh_item(A, item);
      const int ntl = (it.nch + A.cpt - 1) / A.cpt;
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        WT_ACC(w_af, mbar_wait_sleep(&acc_full[buf], use & 1u));
        tc_after();
        const uint32_t col = t_acc + buf * static_cast<uint32_t>(A.Npad) + static_cast<uint32_t>(cb * NC);
        // batches of loads in flight (the register cap does not hold all NC values at once)
#pragma unroll
        for (int j0 = 0; j0 < NC / 4; j0 += NB4) {
          float f[4 * NB4];
#pragma unroll
          for (int j = 0; j < NB4; ++j)
            if (j0 + j < NC / 4) tmem_ld4_nowait(tq + col + 4u * (j0 + j), *reinterpret_cast<float(*)[4]>(f + 4 * j));
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < NB4; ++j)
            if (j0 + j < NC / 4) {
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[4 * (j0 + j) + i] += f[4 * j + i];
            }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        const bool last = tl + 1 == ntl && item + A.G >= A.nitems;
        if (++nacc == flush_tiles || last) flush();
        // after the first tile of item ii the im2col is past item ii - 1: build the pairs of item ii + 1
        if (tl == 0 && item + A.G < A.nitems) fill(ii + 1, item + A.G);
      }
    }
    if (first && t < S2) {  // no tiles: a zero partial
      for (int i = 0; i < nvalid; ++i) gp0[static_cast<size_t>(i) * S2] = 0.0;
    }
    cp_async_wait<0>();
    if (A.dbg && ew == 0 && lane == 0) {
      unsigned long long* o = A.dbg + blockIdx.x * 16;
      o[12] = WT_NOW() - t0; o[13] = w_af;
    }
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int NC>
cudaError_t run_wgrad_h(const CUtensorMap& tm, const WhArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&wgrad_h_kernel<NC>), kWhSmemMax);
  if (e != cudaSuccess) return e;
#ifdef CSC_ROLE_TIMING
  static unsigned long long* dbg = nullptr;
  static int calls = 0;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 16 * 1024);
  cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 16 * 1024, st);
  WhArgs b = a;
  b.dbg = dbg;
  wgrad_h_kernel<NC><<<grid, kWhThreads, smem, st>>>(tm, b);
  if (++calls % 4 == 0) {
    static unsigned long long h[16 * 1024];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost);
    double t[16] = {0};
    for (int bk = 0; bk < grid; ++bk)
      for (int i = 0; i < 16; ++i) t[i] += static_cast<double>(h[bk * 16 + i]) / grid;
    fprintf(stderr,
            "[wgrad_h roles] mma: total %.0f w_accempty %.0f w_bready %.0f w_aready %.0f | tma: total %.0f w_rawempty %.0f | "
            "zconv0: total %.0f w_rawfull %.0f w_bempty %.0f | im2col0: total %.0f w_aempty %.0f fill %.0f | epi0: total %.0f "
            "w_accfull %.0f\n",
            t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], t[9], t[10], t[11], t[12], t[13]);
  }
#else
  wgrad_h_kernel<NC><<<grid, kWhThreads, smem, st>>>(tm, a);
#endif
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- host side
bool wgrad_h_supported(const Geom& g) {
  return g.N > 0 && g.S >= 3 && g.S * g.S <= 128 && g.Wc >= 2 && (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 &&
         static_cast<int64_t>(g.N) * g.K < (int64_t(1) << 31) && tmap_available();
}

WhPlan wgrad_h_plan(const Geom& g, int num_sms) {
  WhPlan p{};
  p.nkg = ceil_div(g.K, 112);
  p.KC = ceil_div(g.K, p.nkg);
  p.Npad = (p.KC + 15) / 16 * 16;
  p.NCH = p.Npad / 16;
  // residual tile pitch: >= Wc + P + 1 (the pair of the last column), == S (mod 32) (the 32 taps of a
  // lane quarter hit 32 banks)
  int pitch = g.Wc + g.P + 1;
  while (pitch % 32 != g.S % 32) ++pitch;
  p.pitch = pitch;
  const int plane = g.Hc * g.Wc;
  const int G = num_sms / p.nkg > 0 ? num_sms / p.nkg : 1;
  const int64_t total = static_cast<int64_t>(g.N > 0 ? g.N : 1) * plane;
  // rows of an item of len positions starting anywhere in a code row, plus the P halo rows
  auto rows_for = [&](int64_t len) { return static_cast<int>((len + 2 * g.Wc - 2) / g.Wc) + g.P; };
  const int bbytes = p.Npad * 128;
  // items: (image, segment of L positions), L a multiple of 64, ~24 items per CTA
  int64_t L = total / (24 * static_cast<int64_t>(G));
  L = (L + 63) / 64 * 64;
  if (L < 256) L = 256;
  if (L > 4096) L = 4096;
  const int rawbytes = p.KC * 64 * 4;
  auto smem_for = [&](int nb, int nr, int64_t len) {
    return 1024 + 2 * nb * bbytes + nr * rawbytes + 5 * rows_for(len) * pitch * 4;
  };
  // raw slots first (bytes in flight), then B stages; shorter items when nothing else fits
  int nb = 2, nr = 3;
  while (nr < 4 && smem_for(nb, nr + 1, L) <= kWhSmemMax) ++nr;
  while (nb < 4 && smem_for(nb + 1, nr, L) <= kWhSmemMax) ++nb;
  while (L > 64 && smem_for(nb, nr, L) > kWhSmemMax) L -= 64;
  // the segment length among those with the same staged residual rows (same shared memory): the smallest
  // busiest-CTA load under the round-robin item order, in chunks + 2 per item (the residual staging); at
  // config 3 L = 832 -> 960: the busiest CTA 360 -> 340 chunk units
  if (g.N > 0) {
    auto load = [&](int64_t len) {
      const int64_t ns = (plane + len - 1) / len;
      const int64_t ni = static_cast<int64_t>(g.N) * ns;
      const int64_t Gi = std::min<int64_t>(G, ni);
      // CTA c takes items c, c + Gi, ...
      std::vector<int64_t> ld(static_cast<size_t>(Gi), 0);
      for (int64_t i = 0; i < ni; ++i) {
        const int64_t sg = i % ns, l = std::min<int64_t>(len, plane - sg * len);
        ld[static_cast<size_t>(i % Gi)] += (l + kWhChunk - 1) / kWhChunk + 2;
      }
      int64_t mx = 0;
      for (int64_t v : ld) mx = std::max(mx, v);
      return mx;
    };
    const int rows0 = rows_for(L);
    int64_t bestL = L, best = load(L);
    for (int64_t l2 = 256; l2 <= 4096; l2 += 64) {
      if (rows_for(l2) > rows0) continue;
      const int64_t c = load(l2);
      if (c < best || (c == best && l2 > bestL)) {
        best = c;
        bestL = l2;
      }
    }
    L = bestL;
  }
  p.NB = nb;
  p.NR = nr;
  p.L = static_cast<int>(L);
  p.rs_rows = rows_for(L);
  p.rs_floats = p.rs_rows * pitch;
  p.nseg = ceil_div(plane, p.L);
  p.nitems = g.N * p.nseg;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_for(nb, nr, L);
  p.cpt = 2;  // 128 positions per accumulator tile (longer tensor-core accumulations lose accuracy: measured)
  {
    const char* ev = std::getenv("CSC_WH_CPT");
    if (ev != nullptr && std::atoi(ev) >= 1 && std::atoi(ev) <= 4) p.cpt = std::atoi(ev);
  }
  p.ok = p.smem <= kWhSmemMax && p.NB >= 2 && p.NR >= 2 && p.KC <= 256;
  return p;
}

cudaError_t launch_wgrad_h(const Geom& g, const WhPlan& p, TmapCache* tmc, const float* z, const float* r,
                           const uint32_t* zmax, const uint32_t* rmax, double* gpart, cudaStream_t st) {
  const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
  cudaError_t e0 = tmap_2d(*tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K, plane * 4,
                           kWhChunk, static_cast<uint32_t>(p.KC), CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (e0 != cudaSuccess) return e0;
  const CUtensorMap& tm = tmc->map;
  WhArgs a{};
  a.r = r;
  a.zmax = zmax;
  a.rmax = rmax;
  a.gpart = gpart;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.Npad = p.Npad; a.NCH = p.NCH; a.nkg = p.nkg; a.G = p.G;
  a.L = p.L; a.nseg = p.nseg; a.nitems = p.nitems;
  a.pitch = p.pitch; a.rs_rows = p.rs_rows; a.rs_floats = p.rs_floats;
  a.NB = p.NB; a.NR = p.NR; a.cpt = p.cpt;
  switch (p.Npad / 4) {
    case 4: return run_wgrad_h<4>(tm, a, p.grid, p.smem, st);
    case 8: return run_wgrad_h<8>(tm, a, p.grid, p.smem, st);
    case 12: return run_wgrad_h<12>(tm, a, p.grid, p.smem, st);
    case 16: return run_wgrad_h<16>(tm, a, p.grid, p.smem, st);
    case 20: return run_wgrad_h<20>(tm, a, p.grid, p.smem, st);
    case 24: return run_wgrad_h<24>(tm, a, p.grid, p.smem, st);
    case 28: return run_wgrad_h<28>(tm, a, p.grid, p.smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csc

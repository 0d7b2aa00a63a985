// csc_wgrad_h.cu -- filter gradient g = Z^T r' on the sm_100a tensor cores at the fp16 rate
// (tcgen05.mma kind::f16, 3-term split, fp32 accumulate), TMA-fed.
//
// Gradient of the Eq.5 fit term (§3.1): for every filter k and tap t = (a, b)
//   g[k][t] = sum_n sum_{(u,v)} z[n,k,u,v] * R_n[(u,v)][t],   R_n[(u,v)][(a,b)] = r'[n, u-P+a, v-P+b]
// (r' = 0 outside the H x W image).  As a GEMM per CTA:  D[t][k] += sum_pos A[t][pos] B[k][pos],
//   M = 128 taps (s^2 <= 121 used), N = Npad filters of one k-group, K = code positions, 16 per MMA.
// Both operands are split after exact power-of-two scalings (reading T6, as csc_conv_h.cu):
//   x_s = x 2^e,  hi = rn11(x_s) (an exact fp16),  lo = fp16_rn(x_s - hi),
//   D += A_hi B_hi + A_hi B_lo + A_lo B_hi   (2^-22 per product, like 3xTF32, at twice its rate).
// e_z from the running bound of max|z| (the code step raises it), e_r from max|r'|.
// Operands:
//   B = z: TMA boxes {64 positions, 16 planes} (fp32, 4 KB) into a ring of raw slots; converter warps
//       write the scaled fp16 hi / lo rows of one 64-position chunk in the canonical K-major SWIZZLE_128B
//       layout (row = filter, 128 B = 64 positions, 16-B chunks XOR row) and release the raw slot at once.
//   A = im2col of r' in TMEM (lane = tap, one 32-bit column = two consecutive positions): the item's
//       residual rows are staged by cp.async, scaled and split once into fp16 PAIRS hp[row][c] =
//       (hi(r[c]), hi(r[c+1])), so a column is one shared load per lane (pitch = s mod 32: the 32 taps of
//       a lane quarter hit 32 banks).
// The accumulator restarts every tile (cpt chunks); the epilogue adds it into fp32 block sums that are
// flushed into the CTA's fp64 partials every kWhFlush tiles, and wgrad_reduce_kernel sums the per-CTA
// partials in a fixed order (deterministic), exactly as csc_wgrad_tc.cu.
//
// CTA (persistent, 28 warps): warp 0 MMA, warp 1 TMA, warps 2..7 z converters (box g -> warp g mod 6),
// warps 8..11 im2col (one per TMEM lane quarter), warps 12..27 epilogue (4 per lane quarter).
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kWhNR = 12;        // raw TMA slots (4 KB each)
constexpr int kWhNA = 4;         // TMEM A slots (64 columns each: 4 K16-steps x (8 hi + 8 lo))
constexpr int kWhZWarps = 6;
constexpr int kWhIWarps = 4;
constexpr int kWhEpiWarps = 16;
constexpr int kWhZBase = 2, kWhIBase = kWhZBase + kWhZWarps, kWhEpiBase = kWhIBase + kWhIWarps;
constexpr int kWhWarps = kWhEpiBase + kWhEpiWarps;
constexpr int kWhThreads = 32 * kWhWarps;
constexpr int kWhRawBytes = 4096;  // {64 positions, 16 planes} fp32
constexpr int kWhChunk = 64;       // positions per chunk (one SW128 atom of fp16 along K)
constexpr int kWhFlush = 32;       // tiles summed in fp32 before each fp64 flush
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

struct WhArgs {
  const float* r;        // [N][H][W]
  const uint32_t* zmax;  // bound on max|z| (float bits)
  const uint32_t* rmax;  // max|r| (float bits)
  double* gpart;         // [G][K][S*S]
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, NCH, nkg, G;
  int L, nseg, nitems;
  int pitch, rs_rows, rs_floats;
  int NB, cpt;
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
  __shared__ __align__(8) uint64_t raw_full[kWhNR], raw_empty[kWhNR];
  __shared__ __align__(8) uint64_t b_ready[8], b_empty[8], a_ready[kWhNA], a_empty[kWhNA], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int bbytes = A.Npad * 128;                       // one of hi / lo of a chunk
  uint8_t* bst = sm;                                     // [NB][hi | lo]
  uint8_t* rawst = bst + 2 * A.NB * bbytes;              // [NR][16][64] fp32
  float* rstage = reinterpret_cast<float*>(rawst + kWhNR * kWhRawBytes);  // [rs_rows][pitch] raw r'
  uint32_t* hp = reinterpret_cast<uint32_t*>(rstage + A.rs_floats);       // hi pairs
  uint32_t* lp = hp + A.rs_floats;                                        // lo pairs
  const int ez = scale_exp_w(*A.zmax), er = scale_exp_w(*A.rmax);

  if (tid == 0) {
    for (int i = 0; i < kWhNR; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], 1);
    }
    for (int i = 0; i < A.NB; ++i) {
      mbar_init(&b_ready[i], A.NCH);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < kWhNA; ++i) {
      mbar_init(&a_ready[i], kWhIWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kWhEpiWarps);
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
    uint32_t cc = 0, tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      const int ntl = (it.nch + A.cpt - 1) / A.cpt;
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_after();
        const uint32_t d = t_acc + buf * static_cast<uint32_t>(A.Npad);
        const int c0 = tl * A.cpt, c1 = min(c0 + A.cpt, it.nch);
        for (int c = c0; c < c1; ++c, ++cc) {
          const uint32_t bs = cc % A.NB, as = cc % kWhNA;
          mbar_wait(&b_ready[bs], (cc / A.NB) & 1u);
          mbar_wait(&a_ready[as], (cc / kWhNA) & 1u);
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
    __syncwarp();
  } else if (warp == 1) {
    // ================================ TMA producer: NCH boxes {64 positions, 16 planes} per chunk
    if (lane == 0) {
      uint32_t g = 0;
      const int plane0 = kg * A.KC;
      for (int item = gi; item < A.nitems; item += A.G) {
        const WhItem it = wh_item(A, item);
        for (int c = 0; c < it.nch; ++c) {
          for (int j = 0; j < A.NCH; ++j, ++g) {
            const uint32_t slot = g % kWhNR, ph = (g / kWhNR) & 1u;
            mbar_wait(&raw_empty[slot], ph ^ 1u);
            mbar_arrive_expect_tx(&raw_full[slot], kWhRawBytes);
            // the inner coordinate p0 + 64 c is a multiple of 4 floats: a 16-B aligned box start; rows past
            // the group (or past the last plane: zero fill) meet D columns the epilogue never reads
            tma_load_2d(su32(rawst + slot * kWhRawBytes), &tmap_z, it.p0 + kWhChunk * c, it.n * A.K + plane0 + 16 * j,
                        &raw_full[slot]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kWhIBase) {
    // ================================ z converters: box g (chunk g / NCH, rows 16 (g % NCH) ..) -> warp g % 6
    // lane i, step s: row k = 2 s + i / 16 of the box, positions 4 (i % 16) .. +3 (one float4, a 512-B
    // warp read per step), written as the 8-B half (i & 1) of the 16-B chunk (i % 16) / 2 of row 16 j + k,
    // swizzled to chunk ((i % 16) / 2) ^ (row & 7)
    const int zw = warp - kWhZBase;
    const float sz = exp2i_w(ez);
    const int cidx = (lane & 15) >> 1, half8 = (lane & 1) * 8;
    uint32_t g = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      const uint32_t ng = static_cast<uint32_t>(it.nch * A.NCH);
      for (uint32_t b = 0; b < ng; ++b, ++g) {
        if (static_cast<int>(g % kWhZWarps) != zw) continue;
        const uint32_t slot = g % kWhNR, ph = (g / kWhNR) & 1u;
        const uint32_t cc = g / A.NCH;  // CTA-wide chunk counter (every item has whole chunks of NCH boxes)
        const int j = static_cast<int>(g % A.NCH);
        const uint32_t bs = cc % A.NB;
        mbar_wait(&raw_full[slot], ph);
        mbar_wait(&b_empty[bs], ((cc / A.NB) & 1u) ^ 1u);  // the MMA is done with the stage's previous chunk
        const uint8_t* rp = rawst + slot * kWhRawBytes;
        uint8_t* hip = bst + bs * 2 * bbytes;
        uint8_t* lop = hip + bbytes;
#pragma unroll 4
        for (int s = 0; s < 8; ++s) {
          const int k = 2 * s + (lane >> 4);
          const float4 x = reinterpret_cast<const float4*>(rp + k * 256)[lane & 15];
          const float a0 = x.x * sz, a1 = x.y * sz, a2 = x.z * sz, a3 = x.w * sz;
          const float h0 = rn11_w(a0), h1 = rn11_w(a1), h2 = rn11_w(a2), h3 = rn11_w(a3);
          const int row = 16 * j + k;
          const int off = row * 128 + ((cidx ^ (row & 7)) << 4) + half8;
          *reinterpret_cast<uint2*>(hip + off) = make_uint2(pack_h2_w(h0, h1), pack_h2_w(h2, h3));
          *reinterpret_cast<uint2*>(lop + off) = make_uint2(pack_h2_w(a0 - h0, a1 - h1), pack_h2_w(a2 - h2, a3 - h3));
        }
        fence_async_shared();  // generic writes before the MMA's async-proxy reads; raw reads before the refill
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&raw_empty[slot]);
          mbar_arrive(&b_ready[bs]);
        }
      }
    }
  } else if (warp < kWhEpiBase) {
    // ================================ im2col: lane = tap t = 32 q + lane, two positions per TMEM column
    const int q = warp - kWhIBase;
    const int it_tid = tid - 32 * kWhIBase;  // 0..127
    const int t = 32 * q + lane;
    const int S2 = A.S * A.S;
    const int ta = t < S2 ? t / A.S : 0, tb = t < S2 ? t - ta * A.S : 0;
    const int toff = ta * A.pitch + tb;  // taps past s^2 read offset 0 (finite; their D rows are never read)
    const uint32_t tq = static_cast<uint32_t>(32 * q) << 16;
    const float sr = exp2i_w(er);
    // rstage[rho][c] = r'[n, u_first - P + rho, c - P] (0 outside the image)
    auto stage = [&](int item) {
      const WhItem it = wh_item(A, item);
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      for (int e = it_tid; e < A.rs_floats; e += 32 * kWhIWarps) {
        const int rho = e / A.pitch, c = e - rho * A.pitch;
        const int i = it.u_first - A.P + rho, jc = c - A.P;
        const bool ok = i >= 0 && i < A.H && jc >= 0 && jc < A.W;
        cp_async4(su32(rstage + e), ok ? rn + static_cast<size_t>(i) * A.W + jc : rn, ok);
      }
      cp_async_commit();
    };
    uint32_t cc = 0;
    if (gi < A.nitems) stage(gi);
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      cp_async_wait<0>();
      named_sync(1, 32 * kWhIWarps);  // the staged rows are complete; every warp is done with the old pairs
      for (int e = it_tid; e < A.rs_floats; e += 32 * kWhIWarps) {
        const float x0 = rstage[e] * sr;
        const float x1 = (e + 1 < A.rs_floats ? rstage[e + 1] : 0.f) * sr;
        const float h0 = rn11_w(x0), h1 = rn11_w(x1);
        hp[e] = pack_h2_w(h0, h1);
        lp[e] = pack_h2_w(x0 - h0, x1 - h1);
      }
      named_sync(1, 32 * kWhIWarps);  // pairs complete; the raw stage is free
      if (item + A.G < A.nitems) stage(item + A.G);
      const uint32_t* sh = hp + toff;
      const uint32_t* sl = lp + toff;
      for (int c = 0; c < it.nch; ++c, ++cc) {
        const uint32_t as = cc % kWhNA;
        mbar_wait_sleep(&a_empty[as], ((cc / kWhNA) & 1u) ^ 1u);
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
    }
    cp_async_wait<0>();
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
    uint32_t tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WhItem it = wh_item(A, item);
      const int ntl = (it.nch + A.cpt - 1) / A.cpt;
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait_sleep(&acc_full[buf], use & 1u);
        tc_after();
        const uint32_t col = t_acc + buf * static_cast<uint32_t>(A.Npad) + static_cast<uint32_t>(cb * NC);
#pragma unroll
        for (int j = 0; j < NC / 4; ++j) {
          float f[4];
          tmem_ld4_nowait(tq + col + 4u * j, f);
          tmem_ld_wait();
          acc[4 * j] += f[0];
          acc[4 * j + 1] += f[1];
          acc[4 * j + 2] += f[2];
          acc[4 * j + 3] += f[3];
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        const bool last = tl + 1 == ntl && item + A.G >= A.nitems;
        if (++nacc == kWhFlush || last) flush();
      }
    }
    if (first && t < S2) {  // no tiles: a zero partial
      for (int i = 0; i < nvalid; ++i) gp0[static_cast<size_t>(i) * S2] = 0.0;
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
  wgrad_h_kernel<NC><<<grid, kWhThreads, smem, st>>>(tm, a);
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
  auto smem_for = [&](int nb, int64_t len) {
    return 1024 + 2 * nb * bbytes + kWhNR * kWhRawBytes + 3 * rows_for(len) * pitch * 4;
  };
  int nb = 4;
  while (nb > 2 && smem_for(nb, L) > kWhSmemMax) --nb;
  while (L > 64 && smem_for(nb, L) > kWhSmemMax) L -= 64;
  p.NB = nb;
  p.L = static_cast<int>(L);
  p.rs_rows = rows_for(L);
  p.rs_floats = p.rs_rows * pitch;
  p.nseg = ceil_div(plane, p.L);
  p.nitems = g.N * p.nseg;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_for(nb, L);
  p.cpt = 1;
  {
    const char* ev = std::getenv("CSC_WH_CPT");
    if (ev != nullptr && std::atoi(ev) >= 1 && std::atoi(ev) <= 4) p.cpt = std::atoi(ev);
  }
  p.ok = p.smem <= kWhSmemMax && p.NB >= 2;
  return p;
}

cudaError_t launch_wgrad_h(const Geom& g, const WhPlan& p, TmapCache* tmc, const float* z, const float* r,
                           const uint32_t* zmax, const uint32_t* rmax, double* gpart, cudaStream_t st) {
  const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
  cudaError_t e0 = tmap_2d(*tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K, plane * 4,
                           kWhChunk, 16, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
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
  a.NB = p.NB; a.cpt = p.cpt;
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

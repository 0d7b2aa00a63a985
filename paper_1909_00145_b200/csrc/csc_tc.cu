// csc_tc.cu -- tensor-core (tcgen05, 3xTF32) dense passes of the CSC hot path on sm_100a.
//
// Dense pass: y[n,i,j] = sum_k sum_{a,b} f[k,a,b] z[n,k,i+P-a,j+P-b]
// is computed as an implicit GEMM followed by a shift-add ("col2im"):
//   Y[pos][tap] = sum_k z[k][pos] * f[k][tap]      M = 128 code positions, N = taps (s^2 padded),
//                                                  K = filters, 8 per tcgen05.mma (kind::tf32)
//   y[i][j]     = sum_{a,b} Y[(i+P-a, j+P-b)][a*s+b]
// 3xTF32: z = z_hi + z_lo, f = f_hi + f_lo (hi = rna_tf32(x), lo = rna_tf32(x - hi));
// Y += z_hi f_hi + z_hi f_lo + z_lo f_hi (z_lo f_lo dropped, ~2^-22 relative, unbiased) --
// plain TF32 fails the 1e-5 parity bar, 3xTF32 keeps it.
//
// CTA = one SM (persistent, 21 warps):
//   warp 0        TMEM allocation + single-thread MMA issue (A from TMEM, B from smem)
//   warps 4..11   epilogue: TMEM -> registers, warp-shuffle sum over the s column taps,
//                 read-modify-write into a per-lane-quarter shared-memory window of output rows
//                 (the two warps of a quarter take disjoint tap rows, so no two warps ever
//                 write the same address and no per-step barrier is needed)
//   warps 12..23  converters: coalesced loads of z (one code position per lane), hi/lo split
//                 (round-to-nearest tf32), tcgen05.st into a 16-slot TMEM ring of A chunks
// B (filter taps of this k-split, hi and lo, MN-major SWIZZLE_128B_BASE32B image prepared by
// tc_bimg_kernel) stays resident in shared memory.  Work item = (image n, band of BR code
// rows); positions are grouped in 32-wide row segments (one per warp quarter, never crossing a
// code row), 4 segments per 128-row MMA tile.  Each band writes its (BR+P) x W window of
// partial output rows; tc_fixup_kernel sums the overlapping windows in a fixed order.
#include "csc_internal.cuh"

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace csc {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kNS = 4;            // TMEM A slots: kKSteps K-steps each, 64 columns (32 hi + 32 lo)
constexpr int kKSteps = 4;        // K-steps (8 filters each) per slot
constexpr int kEpiWarps = 8;      // epilogue warps (2 per TMEM lane quarter, disjoint tap rows)
constexpr int kConvPerQ = 4;        // converter warps per TMEM lane quarter
constexpr int kKPerConv = kKSteps / kConvPerQ;  // K-steps of a slot filled by one converter warp
constexpr int kConvWarps = 4 * kConvPerQ;
constexpr int kEpiBase = 1, kConvBase = kEpiBase + kEpiWarps;
constexpr int kTcWarps = kConvBase + kConvWarps;
constexpr int kTcThreads = 32 * kTcWarps;

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, unsigned long long& acc, bool on) {
  if (!on) { mbar_wait(bar, parity); return; }
  const unsigned long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - t0;
}
// Wait with a suspend-time hint: the warp sleeps in the barrier unit instead of re-issuing
// try_wait, leaving issue slots to the MMA / converter warps sharing its SMSP.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity), "r"(20000)
      : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// SWIZZLE_128B_BASE32B smem descriptor (tf32 MN-major): LBO = MN-atom stride, SBO = K-atom stride.
__device__ __forceinline__ uint64_t sdesc_b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(1) << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
// kind::tf32, fp32 accumulate, A K-major (TMEM), B MN-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32_ts(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// Warp-collective forms: every lane calls, one elected lane issues.
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(bar))
      : "memory");
}

// One K-step of 3xTF32 MMAs (3 products) issued by one elected lane in a single asm block: the
// operand arithmetic stays inside PTX, so the issue loop costs a few instructions per MMA
// instead of an elect + uniform-register moves per MMA.
__device__ __forceinline__ void mma_kstep3(uint32_t d, uint32_t ah, uint64_t bh, uint64_t bl, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n.reg .pred e, p, t;\n.reg .b32 al;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\nadd.u32 al, %1, %6;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], %2, %4, t;\n"
      "}\n" ::"r"(d), "r"(ah), "l"(bh), "l"(bl), "r"(idesc), "r"(acc), "n"(8 * kKSteps)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float (&f)[16]) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&f)[16]) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
}
// 3xTF32 split: hi = rna_tf32(x), lo = rna_tf32(x - hi).  Both are exactly representable in
// tf32, so the tensor core's operand truncation is exact; lo has a random sign relative to x, so
// the dropped lo*lo term (~2^-22 relative) carries no systematic bias.
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  // cvt.rna.tf32.f32 (round to nearest, ties away) written as integer add + mask: identical
  // results for finite x, 2 integer ops instead of the ~5-instruction emulation ptxas emits
  hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  lo = (__float_as_uint(x - __uint_as_float(hi)) + 0x1000u) & 0xFFFFE000u;
}
__device__ __forceinline__ float ldg_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];\n" : "=f"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

struct TcArgs {
  const float* z;
  const float* bimg;  // [nks][2][natoms][KC][32] swizzled
  float* part;        // [nks][N][nbands][BR+P][W]
  double* l1_part;    // [nks * grid] or nullptr
  int N, K, S, H, W, Hc, Wc, P;
  int KC, NCH, NT, natoms, ks;
  int BR, nbands, nitems, SEGR, RW;
  int dbg;  // development switches (CSC_TC_DEBUG): 1 = converters skip loads, 2 = epilogue skips col2im,
            // 4 = MMA issues 1 product instead of 3, 8 = record per-role wait cycles into dbgbuf
  unsigned long long* dbgbuf;  // [grid][8] when dbg & 8
};

struct ItemInfo {
  int n, u0, u1, ntiles;
};
__device__ __forceinline__ ItemInfo decode_item(const TcArgs& A, int item) {
  ItemInfo it;
  it.n = item / A.nbands;
  const int b = item - it.n * A.nbands;
  it.u0 = b * A.BR;
  it.u1 = min(it.u0 + A.BR, A.Hc);
  it.ntiles = (A.SEGR * (it.u1 - it.u0) + 3) / 4;
  return it;
}

// ---------------------------------------------------------------- the dense-pass kernel
template <int S>
__global__ void __launch_bounds__(kTcThreads, 1) conv_tc_kernel(const TcArgs A) {
  constexpr int P = S - 1;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t a_full[kNS], a_empty[kNS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double l1_warp[kConvWarps];

  // warp index broadcast from lane 0: provably warp-uniform, so role-specific values stay in the
  // uniform datapath (no per-MMA R2UR moves in the single-thread MMA issue loop)
  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int bbytes = A.natoms * A.KC * 128;  // one of hi / lo
  uint8_t* bsm = sm;                         // [hi | lo]
  float* ring = reinterpret_cast<float*>(sm + 2 * bbytes);
  const int ring_floats = (A.BR + P) * A.RW;  // one window per lane quarter (4 windows)

  // ---- setup: B image -> smem, ring = 0, barriers, TMEM
  {
    const int4* src = reinterpret_cast<const int4*>(A.bimg + static_cast<size_t>(A.ks) * 2 * A.natoms * A.KC * 32);
    int4* dst = reinterpret_cast<int4*>(bsm);
    for (int e = tid; e < 2 * bbytes / 16; e += kTcThreads) dst[e] = src[e];
    for (int e = tid; e < 4 * ring_floats; e += kTcThreads) ring[e] = 0.f;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&a_full[i], kConvWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);

  if (warp == 0) {
    // ================================ MMA issuer
    // The whole warp runs the loop with warp-uniform values only (no lane-dependent branches), so
    // every operand stays in the uniform datapath; one elected lane issues each tcgen05.mma.
    const uint32_t idesc = idesc_tf32_ts(A.NT);
    const uint32_t lbo = static_cast<uint32_t>(A.KC) * 128u;
    const uint32_t sbh = su32(bsm), sbl = su32(bsm + bbytes);
    uint32_t g = 0, tcount = 0;
    for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
      const ItemInfo it = decode_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_after();
        const uint32_t d = tbase + buf * 128u;
        for (int c0 = 0; c0 < A.NCH; c0 += kKSteps, ++g) {
          const uint32_t slot = g % kNS, ph = (g / kNS) & 1u;
          mbar_wait(&a_full[slot], ph);
          tc_after();
          const int ns = min(kKSteps, A.NCH - c0);
          const uint32_t a0 = tbase + 256u + slot * (16u * kKSteps);
#pragma unroll
          for (int e = 0; e < kKSteps; ++e) {
            if (e < ns) {
              // K-step c0 + e: B start address + (c0 + e) * 1024 B (8 K-rows of 128 B)
              const uint32_t koff = static_cast<uint32_t>(c0 + e) * 1024u;
              const uint64_t bh = sdesc_b32(sbh + koff, lbo, 512u);
              const uint64_t bl = sdesc_b32(sbl + koff, lbo, 512u);
              const uint32_t acc = (c0 + e) > 0 ? 1u : 0u;
              mma_kstep3(d, a0 + e * 8u, bh, bl, idesc, acc);
            }
          }
          mma_commit_elect(&a_empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= kEpiBase && warp < kConvBase) {
    // ================================ epilogue (col2im into the quarter's window)
    const int q = warp & 3;                   // TMEM lane quarter
    const int h = (warp - kEpiBase) >> 2;     // tap-row half (warps 1..4 and 5..8 each cover the 4 quarters)
    constexpr int AH = (S + 1) / 2;
    const int a_beg = h == 0 ? 0 : AH, a_end = h == 0 ? AH : S;
    float* win = ring + q * ring_floats;
    uint32_t tcount = 0;
    unsigned long long w_epi = 0;
    for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
      const ItemInfo it = decode_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        if (A.dbg & 8) mbar_wait_t(&acc_full[buf], use & 1u, w_epi, true);
        else if (A.dbg & 64) mbar_wait(&acc_full[buf], use & 1u);
        else mbar_wait_sleep(&acc_full[buf], use & 1u);
        tc_after();
        const int sg = t * 4 + q;
        const int u = it.u0 + sg / A.SEGR;
        const int v0 = (sg % A.SEGR) * 32;
        const bool seg_ok = u < it.u1;
        const uint32_t tacc = tbase + buf * 128u + (static_cast<uint32_t>(32 * q) << 16);
#pragma unroll 1
        for (int a = a_beg; a < a_end; a += 2) {
          const bool two = a + 1 < a_end;
          float y0[16], y1[16];
          if (A.dbg & 32) continue;
          tmem_ld16_nowait(tacc + a * S, y0);
          if (two) tmem_ld16_nowait(tacc + (a + 1) * S, y1);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          if (!seg_ok || (A.dbg & 2)) continue;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            if (rr == 1 && !two) break;
            const float* y = rr == 0 ? y0 : y1;
            // column sums over the s taps of row a (fixed order: even/odd partial chains)
            float u0s = 0.f, u1s = 0.f, d0s = 0.f, d1s = 0.f;
#pragma unroll
            for (int b = 0; b < S; ++b) {
              const float up = __shfl_up_sync(kFullMask, y[b], b);
              const float dn = __shfl_down_sync(kFullMask, y[b], 32 - b);
              const float uv = lane >= b ? up : 0.f;
              const float dv = (b > 0 && lane < b) ? dn : 0.f;
              if (b & 1) { u1s += uv; d1s += dv; } else { u0s += uv; d0s += dv; }
            }
            float upv[1] = {u0s + u1s}, dnv[1] = {d0s + d1s};
            float* up = upv;
            float* dn = dnv;
            float* row = win + (u - it.u0 + a + rr) * A.RW + v0 + lane;
            row[0] += up[0];
            if (lane < P) row[32] += dn[0];
          }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        named_sync(1 + q, 64);  // the quarter's two warps finish a tile before the next one starts
      }
      // band done: sum the 4 windows into the band's partial (accumulating across k-splits)
      named_sync(5, 32 * kEpiWarps);
      float* dst = A.part + (static_cast<size_t>(it.n) * A.nbands + (it.u0 / A.BR)) *
                                static_cast<size_t>(A.BR + P) * A.W;
      const int rows = A.BR + P;
      const int et = tid - 32 * kEpiBase;
      for (int e = et; e < rows * A.W; e += 32 * kEpiWarps) {
        const int r = e / A.W, j = e - r * A.W;
        const int o = r * A.RW + j + P;
        const float v = ((ring[o] + ring[ring_floats + o]) + ring[2 * ring_floats + o]) + ring[3 * ring_floats + o];
        dst[e] = A.ks == 0 ? v : dst[e] + v;
      }
      named_sync(5, 32 * kEpiWarps);
      for (int e = et; e < 4 * ring_floats; e += 32 * kEpiWarps) ring[e] = 0.f;
      named_sync(5, 32 * kEpiWarps);
    }
    if ((A.dbg & 8) && warp == kEpiBase && lane == 0) A.dbgbuf[blockIdx.x * 8 + 3] = w_epi;
  } else if (warp >= kConvBase) {
    // ================================ converters: z -> (hi, lo) -> TMEM A slots
    const int cw = warp - kConvBase;
    const int q = warp & 3;  // lane quarter
    const int e = cw >> 2;   // fills K-step e of every slot
    const uint32_t tq = tbase + (static_cast<uint32_t>(32 * q) << 16);
    const size_t plane = static_cast<size_t>(A.Hc) * A.Wc;
    const bool want_l1 = A.l1_part != nullptr;
    float l1 = 0.f;
    unsigned long long w_cv = 0;
    // iterate this warp's chunk sequence (every kConvPerQ-th chunk) with a 3-deep register
    // prefetch; all index arithmetic is incremental (no integer division per chunk)
    struct Cur {
      int item, t, j, ntiles, n, u0, u1, urow, scol;
      uint32_t g;
      bool done;
    };
    const int NSL = (A.NCH + kKSteps - 1) / kKSteps;  // slots per tile
    auto set_item = [&](Cur& s) {
      const ItemInfo it = decode_item(A, s.item);
      s.ntiles = it.ntiles; s.n = it.n; s.u0 = it.u0; s.u1 = it.u1;
      s.t = 0;
      s.urow = it.u0 + q / A.SEGR;
      s.scol = q % A.SEGR;
    };
    auto first = [&](Cur& s) {
      s.item = blockIdx.x;
      s.j = 0;
      s.g = 0;
      s.done = s.item >= A.nitems;
      if (!s.done) set_item(s);
    };
    auto advance1 = [&](Cur& s) {  // next slot, incremental index arithmetic only
      ++s.g;
      if (++s.j < NSL) return;
      s.j = 0;
      if (++s.t < s.ntiles) {
        s.scol += 4;
        while (s.scol >= A.SEGR) { s.scol -= A.SEGR; ++s.urow; }
        return;
      }
      s.item += gridDim.x;
      if (s.item >= A.nitems) { s.done = true; return; }
      set_item(s);
    };
    // this warp fills K-steps e, e + kConvPerQ, ... of every slot (kKPerConv of them)
    auto load = [&](const Cur& s, float (&v)[8 * kKPerConv]) {
#pragma unroll
      for (int jj = 0; jj < 8 * kKPerConv; ++jj) v[jj] = 0.f;
      if (s.done) return;
      const int vv = s.scol * 32 + lane;
      if (s.urow >= s.u1 || vv >= A.Wc || (A.dbg & 1)) return;
      const float* pb = A.z + static_cast<size_t>(s.n) * A.K * plane + static_cast<size_t>(s.urow) * A.Wc + vv;
#pragma unroll
      for (int m = 0; m < kKPerConv; ++m) {
        const int kk = s.j * kKSteps + e + m * kConvPerQ;
        if (kk >= A.NCH) break;
        const int k0 = A.ks * A.KC + kk * 8;
        const float* p = pb + static_cast<size_t>(k0) * plane;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (k0 + jj < A.K) v[m * 8 + jj] = ldg_stream(p + jj * plane);
      }
    };
    // D-deep prefetch with static buffer indices: buffer i is consumed and immediately refilled
    // with the slot D ahead, so no instruction reads a register whose load is still in flight
    // before its turn (a rotating register ring would stall on every in-flight load).
    constexpr int D = 3;
    Cur cur, pre;
    first(cur);
    pre = cur;
    float v[D][8 * kKPerConv];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      load(pre, v[i]);
      if (!pre.done) advance1(pre);
    }
    while (!cur.done) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if (cur.done) break;
        const uint32_t slot = cur.g % kNS, ph = (cur.g / kNS) & 1u;
        if (A.dbg & 8) mbar_wait_t(&a_empty[slot], ph ^ 1u, w_cv, true);
        else if (A.dbg & 64) mbar_wait(&a_empty[slot], ph ^ 1u);
        else mbar_wait_sleep(&a_empty[slot], ph ^ 1u);
        tc_after();
#pragma unroll
        for (int m = 0; m < kKPerConv; ++m) {
          const int kk = cur.j * kKSteps + e + m * kConvPerQ;
          uint32_t h8[8], l8[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float x = v[i][m * 8 + jj];
            if (A.dbg & 128) {
              h8[jj] = __float_as_uint(x);
              l8[jj] = __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
            } else {
              tf32_split(x, h8[jj], l8[jj]);
            }
            if (want_l1) l1 += fabsf(x);
          }
          if (kk < A.NCH && !(A.dbg & 16)) {
            const uint32_t ta = tq + 256u + slot * (16u * kKSteps) + static_cast<uint32_t>(e + m * kConvPerQ) * 8u;
            tmem_st8(ta, h8);
            tmem_st8(ta + 8u * kKSteps, l8);
          }
        }
        load(pre, v[i]);
        if (!pre.done) advance1(pre);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[slot]);
        advance1(cur);
      }
    }
    if ((A.dbg & 8) && warp == kConvBase && lane == 0) A.dbgbuf[blockIdx.x * 8 + 4] = w_cv;
    const double t = warp_sum_d(static_cast<double>(l1));
    if (lane == 0) l1_warp[cw] = t;
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(512));
  if (tid == 0 && A.l1_part != nullptr) {
    double s = 0.0;
    for (int i = 0; i < kConvWarps; ++i) s += l1_warp[i];
    A.l1_part[static_cast<size_t>(A.ks) * gridDim.x + blockIdx.x] = s;
  }
}

// B image: bimg[ks][hl][atom][k][32 taps] with the SWIZZLE_128B_BASE32B pattern
// (32-byte granule index XOR (k & 3)); hl = 0: raw fp32 (tensor core truncates to tf32),
// hl = 1: x - trunc_tf32(x).
__global__ void tc_bimg_kernel(const float* __restrict__ f, int K, int S2, int KC, int nks, int natoms,
                               float* __restrict__ bimg) {
  const int total = nks * KC * natoms * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int nn = e % 32;
    int r = e / 32;
    const int k = r % KC;
    r /= KC;
    const int atom = r % natoms;
    const int ks = r / natoms;
    const int n = atom * 32 + nn;
    const int kg = ks * KC + k;
    const float v = (kg < K && n < S2) ? f[static_cast<size_t>(kg) * S2 + n] : 0.f;
    const size_t blk = static_cast<size_t>(natoms) * KC * 32;  // floats per (ks, hl)
    const size_t off = static_cast<size_t>(atom) * KC * 32 + static_cast<size_t>(k) * 32 +
                       (((nn >> 3) ^ (k & 3)) << 3) + (nn & 7);
    uint32_t vh, vl;
    tf32_split(v, vh, vl);
    bimg[(static_cast<size_t>(ks) * 2 + 0) * blk + off] = __uint_as_float(vh);
    bimg[(static_cast<size_t>(ks) * 2 + 1) * blk + off] = __uint_as_float(vl);
  }
}

// Sum the overlapping band windows (fixed order: k-split, then band), then
//   residual mode: r = y - x, sq += r^2;   sum-of-squares mode: sq += y^2.
__global__ void tc_fixup_kernel(const float* __restrict__ part, int N, int H, int W, int P, int BR, int nbands,
                                int nks, const float* __restrict__ x, float* __restrict__ r, int mode,
                                double* __restrict__ sq_part) {
  // one output row per block iteration (row index decoded once; threads run along the row)
  const size_t win = static_cast<size_t>(BR + P) * W;
  double sq = 0.0;
  for (int row = blockIdx.x; row < N * H; row += gridDim.x) {
    const int n = row / H, i = row - n * H;
    const int b0 = i / BR;
    int b1 = (i + P) / BR;
    if (b1 > nbands - 1) b1 = nbands - 1;
    const float* pk = part + static_cast<size_t>(n) * nbands * win;
    const size_t orow = static_cast<size_t>(row) * W;
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
      float v = 0.f;
      for (int b = b0; b <= b1; ++b) v += pk[b * win + static_cast<size_t>(i - b * BR + P) * W + j];
      if (mode == kConvResidual) {
        if (x != nullptr) v = v - x[orow + j];
        r[orow + j] = v;
      }
      sq += static_cast<double>(v) * static_cast<double>(v);
    }
  }
  // block reduction (fixed tree)
  __shared__ double red[32];
  double t = sq;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFullMask, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    sq_part[blockIdx.x] = s;
  }
}

// The fixup's reductions in its last block (one launch less per dense pass): the block sums of r^2 ->
// *out_sq, and the ||z||_1 partials of the dense pass (if any) -> *out_l1, each in a fixed order (thread t
// sums partials t, t + blockDim, ... in turn, then the block's tree; deterministic, and the last block no
// longer walks the 592 partials one dependent L2 load at a time); the block counter (zero at allocation)
// is cleared for the next launch.
__device__ double block_sum_fixed(const double* v, int n) {
  __shared__ double red[32];
  double t = 0.0;
  for (int b = threadIdx.x; b < n; b += blockDim.x) t += __ldcg(v + b);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFullMask, t, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__device__ void fixup_finish(const double* sq_part, const FixupSums& fs) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(fs.counter, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double t = block_sum_fixed(sq_part, static_cast<int>(gridDim.x));
  if (threadIdx.x == 0) *fs.out_sq = t;
  if (fs.l1_part != nullptr) {
    const double u = block_sum_fixed(fs.l1_part, fs.nl1);
    if (threadIdx.x == 0) *fs.out_l1 = u;
  }
  if (threadIdx.x == 0) *fs.counter = 0ull;
}

// Same as tc_fixup_kernel for W % 4 == 0 with 16-B aligned buffers: a thread takes 4 consecutive
// columns (float4) and the block covers 256 / (W/4) rows at once, so each thread has its loads of
// several rows in flight instead of one dependent chain per element.
__global__ void tc_fixup4_kernel(const float* __restrict__ part, int N, int H, int W, int P, int BR, int nbands,
                                 const float4* __restrict__ x, float4* __restrict__ r, int mode,
                                 double* __restrict__ sq_part, FixupSums fs) {
  const size_t win = static_cast<size_t>(BR + P) * W;
  const int W4 = W / 4;
  const int rpb = blockDim.x / W4 > 0 ? blockDim.x / W4 : 1;  // rows per block step
  const int rr = threadIdx.x / W4, j4 = threadIdx.x - rr * W4;
  double sq = 0.0;
  if (rr < rpb && j4 < W4) {
    // two rows per thread per step with all their loads issued first (a row spans at most two bands
    // when P < BR; a third band, if any, is added after)
    const int stride = gridDim.x * rpb;
    for (int row0 = blockIdx.x * rpb + rr; row0 < N * H; row0 += 2 * stride) {
      float4 v[2], xv[2];
      int rows[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = row0 + h * stride;
        rows[h] = row;
        v[h] = make_float4(0.f, 0.f, 0.f, 0.f);
        xv[h] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < N * H) {
          const int n = row / H, i = row - n * H;
          const int b0 = i / BR;
          int b1 = (i + P) / BR;
          if (b1 > nbands - 1) b1 = nbands - 1;
          const float* pk = part + static_cast<size_t>(n) * nbands * win;
          for (int b = b0; b <= b1; ++b) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(pk + b * win + static_cast<size_t>(i - b * BR + P) * W) + j4);
            v[h].x += t.x; v[h].y += t.y; v[h].z += t.z; v[h].w += t.w;
          }
          if (mode == kConvResidual && x != nullptr) xv[h] = __ldg(x + static_cast<size_t>(row) * W4 + j4);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (rows[h] >= N * H) continue;
        float4 w = v[h];
        if (mode == kConvResidual) {
          w.x -= xv[h].x; w.y -= xv[h].y; w.z -= xv[h].z; w.w -= xv[h].w;
          r[static_cast<size_t>(rows[h]) * W4 + j4] = w;
        }
        sq += static_cast<double>(w.x) * w.x + static_cast<double>(w.y) * w.y + static_cast<double>(w.z) * w.z +
              static_cast<double>(w.w) * w.w;
      }
    }
  }
  __shared__ double red[32];
  double t = sq;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFullMask, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    sq_part[blockIdx.x] = s;
  }
  if (fs.out_sq != nullptr) fixup_finish(sq_part, fs);
}

}  // namespace

// ---------------------------------------------------------------- host side
int tc_ntaps_padded(int S) {
  int nt = S * S;
  const int need = (S - 1) * S + 16;
  if (need > nt) nt = need;
  return (nt + 15) / 16 * 16;
}

bool conv_tc_supported(const Geom& g) {
  return (g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) && g.Wc >= 32 && tc_ntaps_padded(g.S) <= 128;
}

TcPlan conv_tc_plan(const Geom& g, int num_sms) {
  constexpr int kSmemBudget = 210 * 1024;
  TcPlan p{};
  p.NT = tc_ntaps_padded(g.S);
  p.natoms = (p.NT + 31) / 32;
  p.SEGR = ceil_div(g.Wc, 32);
  p.RW = p.SEGR * 32 + 32;
  // band height: ~8 items per SM, 4..64 rows
  const int n = g.N > 0 ? g.N : 1;
  int BR = (g.Hc * n) / (8 * num_sms);
  if (BR < 4) BR = 4;
  if (BR > 64) BR = 64;
  if (BR > g.Hc) BR = g.Hc;
  // filters per k-split: as many as fit beside 4 output windows of at least min(BR, 8) rows
  const int br_min = BR < 8 ? BR : 8;
  const int win_min = 4 * (br_min + g.P) * p.RW * 4;
  int kc_fit = (kSmemBudget - 1024 - win_min) / (2 * p.natoms * 128);
  kc_fit = kc_fit / 8 * 8;
  if (kc_fit > kTcMaxKC) kc_fit = kTcMaxKC;
  if (kc_fit < 8) kc_fit = 8;
  p.nks = ceil_div(g.K, kc_fit);
  p.KC = (ceil_div(g.K, p.nks) + 7) / 8 * 8;
  p.NCH = p.KC / 8;
  const int bsm = 2 * p.natoms * p.KC * 128;
  while (BR > 1 && 1024 + bsm + 4 * (BR + g.P) * p.RW * 4 > kSmemBudget) --BR;
  p.BR = BR;
  p.nbands = ceil_div(g.Hc, BR);
  p.nitems = g.N * p.nbands;
  p.grid = p.nitems < num_sms ? p.nitems : num_sms;
  if (p.grid < 1) p.grid = 1;
  p.smem = 1024 + bsm + 4 * (p.BR + g.P) * p.RW * 4;
  p.part_floats = static_cast<size_t>(g.N) * p.nbands * (p.BR + g.P) * g.W;
  p.bimg_floats = static_cast<size_t>(p.nks) * 2 * p.natoms * p.KC * 32;
  return p;
}

template <int S>
static cudaError_t run_conv_tc(const TcArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&conv_tc_kernel<S>), 220 * 1024);
  if (e != cudaSuccess) return e;
  conv_tc_kernel<S><<<grid, kTcThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_conv_tc(const Geom& g, const TcPlan& p, const float* z, const float* filt, float* bimg,
                           float* part, double* l1_part, cudaStream_t st) {
  tc_bimg_kernel<<<64, 256, 0, st>>>(filt, g.K, g.S * g.S, p.KC, p.nks, p.natoms, bimg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  TcArgs a{};
  a.z = z;
  a.bimg = bimg;
  a.part = part;
  a.l1_part = l1_part;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.NCH = p.NCH; a.NT = p.NT; a.natoms = p.natoms;
  a.BR = p.BR; a.nbands = p.nbands; a.nitems = p.nitems; a.SEGR = p.SEGR; a.RW = p.RW;
  a.dbg = 0;
  a.dbgbuf = nullptr;
  for (int ks = 0; ks < p.nks; ++ks) {
    a.ks = ks;
    switch (g.S) {
      case 5: e = run_conv_tc<5>(a, p.grid, p.smem, st); break;
      case 7: e = run_conv_tc<7>(a, p.grid, p.smem, st); break;
      case 9: e = run_conv_tc<9>(a, p.grid, p.smem, st); break;
      case 11: e = run_conv_tc<11>(a, p.grid, p.smem, st); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tc_bimg(const Geom& g, const TcPlan& p, const float* filt, float* bimg, cudaStream_t st) {
  tc_bimg_kernel<<<64, 256, 0, st>>>(filt, g.K, g.S * g.S, p.KC, p.nks, p.natoms, bimg);
  return cudaGetLastError();
}

cudaError_t launch_conv_tc_fixup(const Geom& g, const TcPlan& p, const float* part, const float* x, float* r,
                                 int mode, double* sq_part, cudaStream_t st, const FixupSums* fsum) {
  if (g.W % 4 == 0 && g.W <= 1024 && (reinterpret_cast<uintptr_t>(part) & 15u) == 0 &&
      (x == nullptr || (reinterpret_cast<uintptr_t>(x) & 15u) == 0) &&
      (r == nullptr || (reinterpret_cast<uintptr_t>(r) & 15u) == 0)) {
    tc_fixup4_kernel<<<kFinalizeBlocks, 256, 0, st>>>(part, g.N, g.H, g.W, g.P, p.BR, p.nbands,
                                                       reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(r),
                                                       mode, sq_part, fsum ? *fsum : FixupSums{});
  } else {
    tc_fixup_kernel<<<kFinalizeBlocks, 256, 0, st>>>(part, g.N, g.H, g.W, g.P, p.BR, p.nbands, p.nks, x, r, mode,
                                                      sq_part);
    if (fsum != nullptr) {
      cudaError_t e = launch_reduce_sum(sq_part, kFinalizeBlocks, fsum->out_sq, 1.0, st);
      if (e != cudaSuccess) return e;
      if (fsum->l1_part != nullptr) return launch_reduce_sum(fsum->l1_part, fsum->nl1, fsum->out_l1, 1.0, st);
    }
  }
  return cudaGetLastError();
}

}  // namespace csc

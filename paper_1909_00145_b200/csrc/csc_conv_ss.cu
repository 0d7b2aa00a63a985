// csc_conv_ss.cu -- dense pass y = sum_k f_k * z_k on the sm_100a tensor cores with TMA-fed,
// shared-memory A operands (tcgen05 "SS" MMA, 3xTF32).
//
// Same mathematics as csc_tc.cu (the valid true convolution of Eq.1's fit term):
//   Y[pos][tap] = sum_k z[k][pos] f[k][tap]      M = 128 code positions, N = taps (s^2 padded),
//                                                K = filters, 8 per tcgen05.mma (kind::tf32)
//   y[i][j]     = sum_{a,b} Y[(i+P-a, j+P-b)][a*s+b]      (col2im)
// but the code tile reaches shared memory by TMA instead of through registers:
//   * positions are flattened (p = u*Wc + v) and a band of BR code rows (BR % 4 == 0) starts at a
//     multiple of 4 floats, the 16-byte alignment a TMA box start needs;
//   * one stage = one K-step of one tile: 4 TMA boxes {32 positions, 8 filter planes} with
//     SWIZZLE_128B_ATOM_32B, i.e. the canonical MN-major SW128_BASE32B UMMA layout of A;
//   * 4 converter warps round the stage to tf32 in place (hi = rn_tf32(z)) and write
//     lo = rn_tf32(z - hi) beside it (vectorised shared-memory pass; no TMEM stores);
//   * the MMA reads A hi/lo and B hi/lo (filter taps, resident) from shared memory.
// The epilogue sums the s taps of every tap row with warp shuffles (the flattened index makes the
// row wrap land in the junk columns j >= W) into per-quarter band windows laid out with row pitch
// Wc; tc_fixup_kernel (csc_tc.cu) sums the overlapping windows of neighbouring bands in a fixed
// order, exactly as for the TMEM-fed kernel.
//
// CTA (persistent, 14 warps): warp 0 MMA issue, warp 1 TMA producer, warps 2..5 converters,
// warps 6..13 epilogue (2 per TMEM lane quarter, disjoint tap rows).  Needs Wc >= 128 (one shared
// band window, see the epilogue).
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kSsNS = 12;           // stages (one K-step of one tile each)
constexpr int kSsConvWarps = 4;
constexpr int kSsEpiWarps = 8;
constexpr int kSsConvBase = 2, kSsEpiBase = kSsConvBase + kSsConvWarps;
constexpr int kSsWarps = kSsEpiBase + kSsEpiWarps;
constexpr int kSsThreads = 32 * kSsWarps;
constexpr int kSsStageBytes = 4096;  // 4 atoms x 8 rows x 128 B (one of hi / lo)
constexpr int kSsSmemMax = 220 * 1024;

struct SsArgs {
  const float* bimg;  // [nks][2][natoms][KC][32] swizzled (tc_bimg_kernel)
  float* part;        // [N][nbands][BR+P][W]
  double* l1_part;    // [nks * grid] or nullptr
  int N, K, S, H, W, Hc, Wc, P;
  int KC, NCH, NT, natoms, ks;
  int BR, nbands, nitems, WL;
};

struct SsItem {
  int n, u0, u1, p0, pend, ntiles;
};
__device__ __forceinline__ SsItem ss_item(const SsArgs& A, int item) {
  SsItem it;
  it.n = item / A.nbands;
  const int b = item - it.n * A.nbands;
  it.u0 = b * A.BR;
  it.u1 = min(it.u0 + A.BR, A.Hc);
  it.p0 = it.u0 * A.Wc;
  it.pend = it.u1 * A.Wc;
  it.ntiles = (it.pend - it.p0 + 127) / 128;
  return it;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

template <int S>
__global__ void __launch_bounds__(kSsThreads, 1)
conv_ss_kernel(const __grid_constant__ CUtensorMap tmap_z, const SsArgs A) {
  constexpr int P = S - 1;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t full[kSsNS], ready[kSsNS], empty[kSsNS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double l1_warp[kSsConvWarps];

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int bbytes = A.natoms * A.KC * 128;            // one of hi / lo
  uint8_t* bsm = sm;                                   // [hi | lo]
  uint8_t* stg = sm + 2 * bbytes;                      // [NS][hi 4 KB | lo 4 KB]
  float* win = reinterpret_cast<float*>(stg + kSsNS * 2 * kSsStageBytes);  // [WL]

  // ---- setup: B image -> smem, windows = 0, barriers, TMEM
  {
    const int4* src = reinterpret_cast<const int4*>(A.bimg + static_cast<size_t>(A.ks) * 2 * A.natoms * A.KC * 32);
    int4* dst = reinterpret_cast<int4*>(bsm);
    for (int e = tid; e < 2 * bbytes / 16; e += kSsThreads) dst[e] = src[e];
    for (int e = tid; e < A.WL; e += kSsThreads) win[e] = 0.f;
  }
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kSsNS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&ready[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kSsEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 256);
  if (warp == 1 && lane == 0) tma_prefetch_desc(&tmap_z);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);

  if (warp == 0) {
    // ================================ MMA issuer (warp-uniform loop, one elected lane issues)
    const uint32_t idesc = idesc_tf32(128, A.NT, 1, 1);
    const uint32_t lbo_b = static_cast<uint32_t>(A.KC) * 128u;
    const uint32_t sbh = su32(bsm), sbl = su32(bsm + bbytes), sst = su32(stg);
    uint32_t g = 0, tcount = 0;
    for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
      const SsItem it = ss_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_after();
        const uint32_t d = tbase + buf * 128u;
        for (int c = 0; c < A.NCH; ++c, ++g) {
          const uint32_t slot = g % kSsNS, ph = (g / kSsNS) & 1u;
          mbar_wait(&ready[slot], ph);
          tc_after();
          const uint32_t ah = sst + slot * (2u * kSsStageBytes);
          // A: MN-major, 4 atoms of 32 positions at LBO = 1 KB, K groups of 4 rows at SBO = 512 B
          const uint64_t dah = sdesc(ah, 1024u, 512u, kLayout128B32);
          const uint64_t dal = sdesc(ah + kSsStageBytes, 1024u, 512u, kLayout128B32);
          // B: K-step c = filter rows 8c..8c+7 of the resident image
          const uint64_t dbh = sdesc(sbh + static_cast<uint32_t>(c) * 1024u, lbo_b, 512u, kLayout128B32);
          const uint64_t dbl = sdesc(sbl + static_cast<uint32_t>(c) * 1024u, lbo_b, 512u, kLayout128B32);
          const uint32_t acc0 = c > 0 ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred e, p, t;\n"
              "elect.sync _|e, 0xffffffff;\n"
              "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %3, %4, p;\n"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %6, %4, t;\n"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %4, t;\n"
              "}\n" ::"r"(d),
              "l"(dah), "l"(dal), "l"(dbh), "r"(idesc), "r"(acc0), "l"(dbl)
              : "memory");
          mma_commit_elect(&empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================ TMA producer: 4 boxes {32 positions, 8 planes} per stage
    if (lane == 0) {
      uint32_t g = 0;
      for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
        const SsItem it = ss_item(A, item);
        const int plane0 = it.n * A.K + A.ks * A.KC;
        for (int t = 0; t < it.ntiles; ++t) {
          const int pt = it.p0 + 128 * t;  // multiple of 4 floats (BR % 4 == 0): 16-B aligned box start
          for (int c = 0; c < A.NCH; ++c, ++g) {
            const uint32_t slot = g % kSsNS, ph = (g / kSsNS) & 1u;
            mbar_wait(&empty[slot], ph ^ 1u);
            mbar_arrive_expect_tx(&full[slot], kSsStageBytes);
            const uint32_t dst = su32(stg + slot * (2 * kSsStageBytes));
#pragma unroll
            for (int at = 0; at < 4; ++at)
              tma_load_2d(dst + at * 1024u, &tmap_z, pt + 32 * at, plane0 + 8 * c, &full[slot]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kSsEpiBase) {
    // ================================ converters: stage hi <- rn_tf32(z) in place, lo <- rn_tf32(z - hi)
    // converter warp cw takes every kSsConvWarps-th stage whole (8 float4 per lane), so the
    // warps work on different stages concurrently and a stage's latency is hidden behind the
    // kSsConvWarps - 1 others
    const int cw = warp - kSsConvBase;
    const bool want_l1 = A.l1_part != nullptr;
    double l1 = 0.0;
    uint32_t g = 0;
    for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
      const SsItem it = ss_item(A, item);
      for (int t = 0; t < it.ntiles; ++t) {
        const int pt = it.p0 + 128 * t;
        for (int c = 0; c < A.NCH; ++c, ++g) {
          if (static_cast<int>(g % kSsConvWarps) != cw) continue;
          const uint32_t slot = g % kSsNS, ph = (g / kSsNS) & 1u;
          mbar_wait(&full[slot], ph);
          float4* hi4 = reinterpret_cast<float4*>(stg + slot * (2 * kSsStageBytes));
          float4* lo4 = reinterpret_cast<float4*>(stg + slot * (2 * kSsStageBytes) + kSsStageBytes);
          float4 xv[8];
#pragma unroll
          for (int rep = 0; rep < 8; ++rep) xv[rep] = hi4[lane + 32 * rep];
          float s1 = 0.f;
#pragma unroll
          for (int rep = 0; rep < 8; ++rep) {
            const int e = lane + 32 * rep;
            const float4 x = xv[rep];
            float4 h, l;
            tf32_split_rn(x.x, h.x, l.x);
            tf32_split_rn(x.y, h.y, l.y);
            tf32_split_rn(x.z, h.z, l.z);
            tf32_split_rn(x.w, h.w, l.w);
            hi4[e] = h;
            lo4[e] = l;
            if (want_l1) {
              // element (atom, row, 32-B granule, 4 floats): granule index is XOR-swizzled with
              // (row & 3), which keeps the position set of a row; count codes of this band once
              const int at = e >> 6, row = (e >> 3) & 7, gq = e & 7;
              const int pos0 = pt + 32 * at + 4 * ((((gq >> 1) ^ (row & 3)) << 1) | (gq & 1));
              const int k = A.ks * A.KC + 8 * c + row;
              if (k < A.K) {
                if (pos0 + 0 < it.pend) s1 += fabsf(x.x);
                if (pos0 + 1 < it.pend) s1 += fabsf(x.y);
                if (pos0 + 2 < it.pend) s1 += fabsf(x.z);
                if (pos0 + 3 < it.pend) s1 += fabsf(x.w);
              }
            }
          }
          if (want_l1) l1 += static_cast<double>(s1);
          fence_async_shared();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ready[slot]);
        }
      }
    }
    const double tsum = warp_sum_d(l1);
    if (lane == 0) l1_warp[warp - kSsConvBase] = tsum;
  } else {
    // ================================ epilogue (col2im into the band window)
    // One window for the 4 quarters: within a tile, the "up" sums of different (quarter, tap row)
    // land on distinct window elements when Wc >= 128 (two positions of a tile are < 128 apart, so
    // p + a Wc = p' + a' Wc forces p = p', a = a').  The P halo sums ("dn") of quarter q overlap the
    // "up" sums of quarter q + 1, so they are added in a second phase after a barrier, and a second
    // barrier keeps tiles strictly ordered.
    const int q = warp & 3;                      // TMEM lane quarter
    const int h = (warp - kSsEpiBase) >> 2;      // tap-row half
    constexpr int AH = (S + 1) / 2;
    const int a_beg = h == 0 ? 0 : AH;
    const int na = h == 0 ? AH : S - AH;
    uint32_t tcount = 0;
    for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
      const SsItem it = ss_item(A, item);
      for (int t = 0; t < it.ntiles; ++t, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait_sleep(&acc_full[buf], use & 1u);
        tc_after();
        const int pq = 128 * t + 32 * q;                // segment start relative to the band
        const bool pvalid = it.p0 + pq + lane < it.pend;  // positions past the band belong to the next item
        const uint32_t tacc = tbase + buf * 128u + (static_cast<uint32_t>(32 * q) << 16);
        // window index of output (p - (P-a) Wc - (P-b)) is (p - band start) + a Wc + b; the b-sum
        // leaves it at (p_lane - band start) + a Wc ("up") and + 32 for the halo ("dn")
        float* rowb = win + pq + lane + a_beg * A.Wc;
        float dnv[AH];
#pragma unroll
        for (int i = 0; i < AH; ++i) {
          dnv[i] = 0.f;
          if (i >= na) continue;
          const int a = a_beg + i;
          float y[16];
          tmem_ld16_nowait(tacc + a * S, y);
          tmem_ld_wait();
          float u0s = 0.f, u1s = 0.f, d0s = 0.f, d1s = 0.f;
#pragma unroll
          for (int b = 0; b < S; ++b) {
            const float yv = pvalid ? y[b] : 0.f;
            const float up = __shfl_up_sync(kFullMask, yv, b);
            const float dn = __shfl_down_sync(kFullMask, yv, 32 - b);
            const float uv = lane >= b ? up : 0.f;
            const float dv = (b > 0 && lane < b) ? dn : 0.f;
            if (b & 1) { u1s += uv; d1s += dv; } else { u0s += uv; d0s += dv; }
          }
          rowb[i * A.Wc] += u0s + u1s;
          dnv[i] = d0s + d1s;
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        named_sync(1, 32 * kSsEpiWarps);
        if (lane < P) {
#pragma unroll
          for (int i = 0; i < AH; ++i)
            if (i < na) rowb[i * A.Wc + 32] += dnv[i];
        }
        named_sync(1, 32 * kSsEpiWarps);
      }
      // band done: window element e >= P is output row (u0 - P) + (e - P) / Wc, column (e - P) % Wc
      float* dst = A.part + (static_cast<size_t>(it.n) * A.nbands + (it.u0 / A.BR)) *
                                static_cast<size_t>(A.BR + P) * A.W;
      const int rows = A.BR + P;
      const int et = tid - 32 * kSsEpiBase;
      for (int e = et; e < rows * A.W; e += 32 * kSsEpiWarps) {
        const int r = e / A.W, j = e - r * A.W;
        const float v = win[r * A.Wc + j + P];
        dst[e] = A.ks == 0 ? v : dst[e] + v;
      }
      named_sync(1, 32 * kSsEpiWarps);
      for (int e = et; e < A.WL; e += 32 * kSsEpiWarps) win[e] = 0.f;
      named_sync(1, 32 * kSsEpiWarps);
    }
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) tmem_dealloc(tbase, 256);
  if (tid == 0 && A.l1_part != nullptr) {
    double s = 0.0;
    for (int i = 0; i < kSsConvWarps; ++i) s += l1_warp[i];
    A.l1_part[static_cast<size_t>(A.ks) * gridDim.x + blockIdx.x] = s;
  }
}

template <int S>
cudaError_t run_conv_ss(const CUtensorMap& tm, const SsArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&conv_ss_kernel<S>), kSsSmemMax);
  if (e != cudaSuccess) return e;
  conv_ss_kernel<S><<<grid, kSsThreads, smem, st>>>(tm, a);
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- host side
bool conv_ss_supported(const Geom& g) {
  return (g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) && g.N > 0 && g.Wc >= 128 &&
         (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 && tc_ntaps_padded(g.S) <= 128 && tmap_available();
}

// Fills the fields of p the SS kernel uses (KC, NCH, nks, natoms, NT, BR, nbands, nitems, grid,
// smem, WL, part_floats, bimg_floats); BR is a multiple of 4.
bool conv_ss_plan(const Geom& g, int num_sms, TcPlan& p) {
  p = TcPlan{};
  p.NT = tc_ntaps_padded(g.S);
  p.natoms = (p.NT + 31) / 32;
  const int stages = kSsNS * 2 * kSsStageBytes;
  // band height: ~6 items per SM, multiple of 4
  const int n = g.N > 0 ? g.N : 1;
  int BR = (g.Hc * n) / (6 * num_sms);
  BR = (BR / 4) * 4;
  if (BR < 4) BR = 4;
  if (BR > 32) BR = 32;
  auto wl = [&](int br) { return (br + g.P) * g.Wc + 192; };
  // filters per k-split: as many as fit beside the stages and 4 windows of 4 rows
  int kc_fit = (kSsSmemMax - 2048 - stages - wl(4) * 4) / (2 * p.natoms * 128);
  kc_fit = kc_fit / 8 * 8;
  if (kc_fit > kTcMaxKC) kc_fit = kTcMaxKC;
  if (kc_fit < 8) return false;
  p.nks = ceil_div(g.K, kc_fit);
  p.KC = (ceil_div(g.K, p.nks) + 7) / 8 * 8;
  p.NCH = p.KC / 8;
  const int bsm = 2 * p.natoms * p.KC * 128;
  while (BR > 4 && 2048 + bsm + stages + wl(BR) * 4 > kSsSmemMax) BR -= 4;
  if (2048 + bsm + stages + wl(BR) * 4 > kSsSmemMax) return false;
  p.BR = BR;
  p.WL = wl(BR);
  p.nbands = ceil_div(g.Hc, BR);
  p.nitems = g.N * p.nbands;
  p.grid = p.nitems < num_sms ? p.nitems : num_sms;
  if (p.grid < 1) p.grid = 1;
  p.smem = 1024 + bsm + stages + p.WL * 4;
  p.part_floats = static_cast<size_t>(g.N) * p.nbands * (p.BR + g.P) * g.W;
  p.bimg_floats = static_cast<size_t>(p.nks) * 2 * p.natoms * p.KC * 32;
  p.ss = true;
  return true;
}

cudaError_t launch_conv_ss(const Geom& g, const TcPlan& p, TmapCache* tmc, const float* z, const float* bimg,
                           float* part, double* l1_part, cudaStream_t st) {
  const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
  cudaError_t e0 = tmap_2d(*tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K, plane * 4,
                           32, 8, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (e0 != cudaSuccess) return e0;
  const CUtensorMap& tm = tmc->map;
  SsArgs a{};
  a.bimg = bimg;
  a.part = part;
  a.l1_part = l1_part;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.NCH = p.NCH; a.NT = p.NT; a.natoms = p.natoms;
  a.BR = p.BR; a.nbands = p.nbands; a.nitems = p.nitems; a.WL = p.WL;
  for (int ks = 0; ks < p.nks; ++ks) {
    a.ks = ks;
    cudaError_t e;
    switch (g.S) {
      case 5: e = run_conv_ss<5>(tm, a, p.grid, p.smem, st); break;
      case 7: e = run_conv_ss<7>(tm, a, p.grid, p.smem, st); break;
      case 9: e = run_conv_ss<9>(tm, a, p.grid, p.smem, st); break;
      case 11: e = run_conv_ss<11>(tm, a, p.grid, p.smem, st); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace csc

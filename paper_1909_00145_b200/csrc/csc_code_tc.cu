// csc_code_tc.cu -- masked proximal-gradient code step on the sm_100a tensor cores (tcgen05, 3xTF32),
// "dense-then-mask".
//
// Eq.3-4 (§3.1) with one gradient step (reading R1) and the point-wise shrinkage of
// P:311-312:  for every masked code (k, u, v) of image n (mask M^t, Eq.2, R4/R5; unmasked codes are
// left untouched, R2 / P:260-262)
//   c = sum_{a,b} d[k,a,b] r[n, u-P+a, v-P+b]          (D^T r, r = 0 outside the image)
//   z <- S_{tau lambda}(z - tau c),   S(w, kappa) = sign(w) max(|w| - kappa, 0)  (+0.0 on the dead zone)
// The correlation is computed for all codes as a GEMM per 128-position tile:
//   C[p][k] = sum_t R[p][t] d[k][t]        M = 128 flattened code positions, N = Npad filters,
//                                          K = 128 taps (s^2 <= 121 used), 16 K-steps of 8
// 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi, RN splits): the same products the 1e-5 parity needs.
// The epilogue streams every code of the tile (coalesced loads issued before the MMA completes),
// applies the mask, the step and the shrinkage, and stores only codes whose value changes.
// At p <= 0.5 the z stream (read all, write the changed sectors) is what HBM must move; the
// tensor work is p-independent ("TC dense-then-mask").
//
// Operands:
//   A = im2col of r in TMEM (lane = position, column = tap), built by the converter warps from a
//       zero-padded residual tile in shared memory (cp.async staging, as in csc_wgrad_tc.cu).
//   B = the filters, K-major SWIZZLE_128B in shared memory, hi and lo, resident for the whole CTA.
// CTA (persistent, 25 warps): warp 0 MMA issue; warps 1..8 converters; warps 9..24 epilogue
// (4 per TMEM lane quarter, Npad/4 filters each).
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kCtNS = 4;          // A slots (4 K-steps = 32 taps each) in TMEM
constexpr int kCtConvWarps = 8;
constexpr int kCtEpiWarps = 16;
constexpr int kCtConvBase = 1, kCtEpiBase = kCtConvBase + kCtConvWarps;
constexpr int kCtWarps = kCtEpiBase + kCtEpiWarps;
constexpr int kCtThreads = 32 * kCtWarps;
constexpr int kCtTile = 128;      // positions per tile
constexpr int kCtSmemMax = 220 * 1024;

struct CtArgs {
  const float* r;        // [N][H][W]
  const float* d;        // [K][S][S]
  float* z;              // [N][K][Hc][Wc]
  const uint32_t* mask;  // selection words [nkg*4][plane]: bit i = mask(k = kg*KC + cb*NC + i, p); nullptr = all
  const float* tau;      // device scalar
  uint32_t* zmax;        // bound of max|z| raised by every written code (float bits), or nullptr
  float lam;
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, nkg, G;
  int L, nseg, nitems;   // item = (image, segment of L flattened positions, L % 128 == 0)
  int pitch, rs_rows, rs_floats;
  int b_bytes;           // one of hi / lo: 4 K-atoms x Npad rows x 128 B
  int tau_stride;        // 0: tau[0] for every filter; 1: tau[k] per filter (ESO rule)
};

struct CtItem {
  int n, p0, p1, ntiles, u_first;
};
__device__ __forceinline__ CtItem ct_item(const CtArgs& A, int item) {
  CtItem it;
  it.n = item / A.nseg;
  const int sg = item - it.n * A.nseg;
  it.p0 = sg * A.L;
  it.p1 = min(it.p0 + A.L, A.Hc * A.Wc);
  it.ntiles = (it.p1 - it.p0 + kCtTile - 1) / kCtTile;
  it.u_first = it.p0 / A.Wc;
  return it;
}

template <int S, int NC>
__global__ void __launch_bounds__(kCtThreads, 1) code_tc_kernel(const CtArgs A) {
  constexpr int S2 = S * S;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t a_full[kCtNS], a_empty[kCtNS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  uint8_t* bh = sm;                     // [4 K-atoms][Npad][128 B] hi
  uint8_t* bl = sm + A.b_bytes;         // lo
  float* rs = reinterpret_cast<float*>(sm + 2 * A.b_bytes);  // [2][rs_rows][pitch]

  // ---- setup: filters of this k-group -> K-major SW128 hi/lo images (RN splits)
  for (int e = tid; e < A.Npad * 128; e += kCtThreads) {
    const int k = e >> 7, t = e & 127;
    const int kk = kg * A.KC + k;
    const float v = (k < A.KC && kk < A.K && t < S2) ? A.d[static_cast<size_t>(kk) * S2 + t] : 0.f;
    float h, l;
    tf32_split_rn(v, h, l);
    const int ka = t >> 5, w = t & 31;
    const uint32_t off = static_cast<uint32_t>(ka * A.Npad * 128 + k * 128 + ((((w >> 2) ^ (k & 7))) << 4) + (w & 3) * 4);
    *reinterpret_cast<float*>(bh + off) = h;
    *reinterpret_cast<float*>(bl + off) = l;
  }
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kCtNS; ++i) {
      mbar_init(&a_full[i], kCtConvWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kCtEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  const uint32_t t_acc = tbase;         // 2 x Npad columns
  const uint32_t t_a = tbase + 256u;    // kCtNS slots x 64 columns

  if (warp == 0) {
    // ================================ MMA issuer
    const uint32_t idesc = idesc_tf32(128, A.Npad, 0, 0);
    const uint32_t sbh = su32(bh), sbl = su32(bl);
    const uint32_t katom = static_cast<uint32_t>(A.Npad) * 128u;
    uint32_t g = 0, tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const CtItem it = ct_item(A, item);
      for (int tl = 0; tl < it.ntiles; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_after();
        const uint32_t dcol = t_acc + buf * static_cast<uint32_t>(A.Npad);
        for (int j = 0; j < 4; ++j, ++g) {  // 4 slots of 4 K-steps (32 taps)
          const uint32_t slot = g % kCtNS, ph = (g / kCtNS) & 1u;
          mbar_wait(&a_full[slot], ph);
          tc_after();
          const uint32_t ah = t_a + slot * 64u;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint64_t dbh = sdesc(sbh + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint64_t dbl = sdesc(sbl + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint32_t acc0 = (j > 0 || e > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred e, p, t;\n"
                "elect.sync _|e, 0xffffffff;\n"
                "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, p;\n"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %4, t;\n"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %4, t;\n"
                "}\n" ::"r"(dcol),
                "r"(ah + 8u * e), "r"(ah + 32u + 8u * e), "l"(dbh), "r"(idesc), "r"(acc0), "l"(dbl)
                : "memory");
          }
          mma_commit_elect(&a_empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp < kCtEpiBase) {
    // ================================ converters: im2col(r) -> TMEM (lane = position)
    const int cw = warp - kCtConvBase;  // 0..7
    const int q = warp & 3;
    const int h = cw >> 2;              // K-steps {2h, 2h+1} of every slot
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const int ct = tid - 32 * kCtConvBase;
    auto stage_r = [&](int item, int buf) {
      const CtItem it = ct_item(A, item);
      float* dst = rs + buf * A.rs_floats;
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      for (int e = ct; e < A.rs_floats; e += 32 * kCtConvWarps) {
        const int rho = e / A.pitch, c = e - rho * A.pitch;
        const int i = it.u_first - A.P + rho, j = c - A.P;
        const bool ok = i >= 0 && i < A.H && j >= 0 && j < A.W;
        cp_async4(su32(dst + e), ok ? rn + static_cast<size_t>(i) * A.W + j : rn, ok);
      }
      cp_async_commit();
    };
    // h (K-steps {2h, 2h+1} of every slot) is made a compile-time constant so that every tap
    // offset (t / S) * pitch + t % S below is an immediate
    auto body = [&](auto hc) {
      constexpr int H = decltype(hc)::value;
      uint32_t g = 0;
      int ibuf = 0;
      if (gi < A.nitems) stage_r(gi, 0);
      for (int item = gi; item < A.nitems; item += A.G, ibuf ^= 1) {
        const CtItem it = ct_item(A, item);
        if (item + A.G < A.nitems) stage_r(item + A.G, ibuf ^ 1);
        else cp_async_commit();
        cp_async_wait<1>();
        named_sync(1, 32 * kCtConvWarps);
        const float* rtile = rs + ibuf * A.rs_floats;
        for (int tl = 0; tl < it.ntiles; ++tl) {
          const int p = it.p0 + tl * kCtTile + 32 * q + lane;
          const bool pok = p < it.p1;
          const int u = p / A.Wc, v = p - u * A.Wc;
          // R[p][(a,b)] = r[u-P+a][v-P+b] = rs[u - u_first + a][v + b]
          const float* src = rtile + (pok ? (u - it.u_first) * A.pitch + v : 0);
#pragma unroll
          for (int j = 0; j < 4; ++j, ++g) {  // slot j of the tile: taps 32 j .. 32 j + 31
            const uint32_t slot = g % kCtNS, ph = (g / kCtNS) & 1u;
            mbar_wait_sleep(&a_empty[slot], ph ^ 1u);
            tc_after();
#pragma unroll
            for (int ee = 0; ee < 2; ++ee) {
              const int e = 2 * H + ee;
              uint32_t hv[8], lv[8];
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const int t = 32 * j + 8 * e + jj;
                const float x = (t < S2 && pok) ? src[(t / S) * A.pitch + (t % S)] : 0.f;
                float hf, lf;
                tf32_split_rn(x, hf, lf);
                hv[jj] = __float_as_uint(hf);
                lv[jj] = __float_as_uint(lf);
              }
              const uint32_t col = t_a + slot * 64u + 8u * e;
              tmem_st8(tq + col, hv);
              tmem_st8(tq + col + 32u, lv);
            }
            tmem_st_wait();
            tc_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[slot]);
          }
        }
        named_sync(1, 32 * kCtConvWarps);
      }
    };
    if (h == 0) body(std::integral_constant<int, 0>{});
    else body(std::integral_constant<int, 1>{});
    cp_async_wait<0>();
  } else {
    // ================================ epilogue: z <- S(z - tau c) on masked codes
    const int ew = warp - kCtEpiBase;  // 0..15
    const int q = warp & 3;
    const int cb = ew >> 2;            // filter block of NC
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const float tau = *A.tau;
    const float kappa = tau * A.lam;
    const size_t plane = static_cast<size_t>(A.Hc) * A.Wc;
    const int k0 = kg * A.KC + cb * NC;  // first filter of this warp
    const int kend = min(kg * A.KC + A.KC, A.K);
    float wmax = 0.f;  // largest |code| this thread writes
    uint32_t tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const CtItem it = ct_item(A, item);
      for (int tl = 0; tl < it.ntiles; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        const int pw = it.p0 + tl * kCtTile + 32 * q;  // first position of this quarter (multiple of 32)
        const int p = pw + lane;
        const bool pok = p < it.p1;
        // prefetch the codes of this tile while the MMA runs
        float zv[NC];
        float* zb = A.z + (static_cast<size_t>(it.n) * A.K + k0) * plane + p;
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const bool ok = pok && (k0 + i) < kend;
          zv[i] = ok ? zb[static_cast<size_t>(i) * plane] : 0.f;
        }
        // selection word of this position: bit i = mask(k0 + i, p) (coalesced, L2-resident)
        const uint32_t sel = A.mask == nullptr ? (pok ? 0xffffffffu : 0u)
                                               : (pok ? __ldg(A.mask + static_cast<size_t>(kg * 4 + cb) * plane + p) : 0u);
        mbar_wait_sleep(&acc_full[buf], use & 1u);
        tc_after();
        const uint32_t colb = t_acc + buf * static_cast<uint32_t>(A.Npad) + static_cast<uint32_t>(cb * NC);
        auto epi = [&](auto per_k) {
          constexpr bool PK = decltype(per_k)::value;
#pragma unroll
          for (int j4 = 0; j4 < NC / 4; ++j4) {
            float c4[4];
            tmem_ld4_nowait(tq + colb + 4u * j4, c4);
            tmem_ld_wait();
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const int i = 4 * j4 + i4;
              const float tk = PK ? __ldg(A.tau + min(k0 + i, A.K - 1)) : tau;
              const float kk = PK ? tk * A.lam : kappa;
              const float w = fmaf(-tk, c4[i4], zv[i]);
              const float nz = w - fminf(fmaxf(w, -kk), kk);  // S_kk(w): w -/+ kk outside [-kk, kk], +0 inside
              if (((sel >> i) & 1u) && (k0 + i) < kend && nz != zv[i]) {
                zb[static_cast<size_t>(i) * plane] = nz;
                wmax = fmaxf(wmax, fabsf(nz));
              }
            }
          }
        };
        if (A.tau_stride) epi(std::true_type{});
        else epi(std::false_type{});
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
    }
    uint32_t wb = __float_as_uint(wmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wb = max(wb, __shfl_xor_sync(kFullMask, wb, o));
    if (lane == 0 && A.zmax != nullptr && wb != 0u) atomicMax(A.zmax, wb);
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// Selection-word mask layout for the tensor-core code step: one 32-bit word per (filter block,
// position), the block being the NC filters one epilogue warp owns:
//   sw[(kg*4 + cb)][p] bit i = mask(k, u, v),  k = kg*KC + cb*NC + i,  p = u*Wc + v,
// with the canonical index l = (k*Hc + u)*Wc + v = k*Hc*Wc + p, Philox block l >> 2, word l & 3
// (#13).  A thread makes 4 consecutive positions of one block: each Philox call of a
// filter yields the 4 positions' words when l is 4-aligned.
constexpr uint32_t kMaskTag = 0x4353434Du;
constexpr uint32_t kSectorTag = 0x43534253u;  // block-structured masks (E5)
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ uint32_t word_of(const uint4& b, int i) {
  return i == 0 ? b.x : (i == 1 ? b.y : (i == 2 ? b.z : b.w));
}
__global__ void mask_selwords_kernel(int K, int KC, int NC, int nper, int nblk, int64_t plane, uint64_t seed,
                                     uint32_t iter, const uint32_t* __restrict__ iter_off, uint64_t thr, int mode,
                                     uint32_t* __restrict__ sw) {
  if (iter_off != nullptr) iter += *iter_off;  // device-side step counter (CUDA-graph replays)
  const int64_t nq = (plane + 3) / 4;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<int64_t>(nblk) * nq) return;
  const int blk = static_cast<int>(tid / nq);
  const int64_t p0 = (tid - static_cast<int64_t>(blk) * nq) * 4;
  const int kg = blk / nper, cb = blk - kg * nper;
  const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  uint32_t out[4] = {0u, 0u, 0u, 0u};
  const int nvalid = min(NC, min(KC - cb * NC, K - kg * KC - cb * NC));  // filters of this word
  // the filters' Philox draws are independent: unrolled, several 10-round chains are in flight at once
#pragma unroll 4
  for (int i = 0; i < nvalid; ++i) {
    const int k = kg * KC + cb * NC + i;
    const uint64_t l0 = static_cast<uint64_t>(k) * plane + p0;
    if (mode == 1) {
      // block-structured masks (E5): one draw per aligned 8-coordinate block b = l >> 3
      const uint64_t qa = (l0 >> 3) >> 2, qb = ((l0 + 3) >> 3) >> 2;
      const uint4 ba = philox4x32_10(make_uint4(static_cast<uint32_t>(qa), static_cast<uint32_t>(qa >> 32), iter, kSectorTag), key);
      const uint4 bb = qb != qa ? philox4x32_10(make_uint4(static_cast<uint32_t>(qb), static_cast<uint32_t>(qb >> 32), iter,
                                                           kSectorTag), key)
                                : ba;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t b = (l0 + j) >> 3;
        const uint32_t rnd = word_of((b >> 2) == qa ? ba : bb, static_cast<int>(b & 3));
        if (static_cast<uint64_t>(rnd) < thr) out[j] |= 1u << i;
      }
      continue;
    }
    const uint64_t qa = l0 >> 2;
    const uint4 ba = philox4x32_10(make_uint4(static_cast<uint32_t>(qa), static_cast<uint32_t>(qa >> 32), iter, kMaskTag), key);
    uint4 bb = ba;
    if ((l0 & 3) != 0)
      bb = philox4x32_10(make_uint4(static_cast<uint32_t>(qa + 1), static_cast<uint32_t>((qa + 1) >> 32), iter, kMaskTag), key);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t l = l0 + j;
      const uint32_t rnd = (l >> 2) == qa ? word_of(ba, static_cast<int>(l & 3)) : word_of(bb, static_cast<int>(l & 3));
      if (static_cast<uint64_t>(rnd) < thr) out[j] |= 1u << i;
    }
  }
  uint32_t* dst = sw + static_cast<int64_t>(blk) * plane + p0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (p0 + j < plane) dst[j] = out[j];
}

template <int S, int NC>
cudaError_t run_code_tc(const CtArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&code_tc_kernel<S, NC>), kCtSmemMax);
  if (e != cudaSuccess) return e;
  code_tc_kernel<S, NC><<<grid, kCtThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int S>
cudaError_t run_code_tc_nc(const CtArgs& a, int grid, int smem, cudaStream_t st) {
  switch (a.Npad / 4) {
    case 4: return run_code_tc<S, 4>(a, grid, smem, st);
    case 8: return run_code_tc<S, 8>(a, grid, smem, st);
    case 12: return run_code_tc<S, 12>(a, grid, smem, st);
    case 16: return run_code_tc<S, 16>(a, grid, smem, st);
    case 20: return run_code_tc<S, 20>(a, grid, smem, st);
    case 24: return run_code_tc<S, 24>(a, grid, smem, st);
    case 28: return run_code_tc<S, 28>(a, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// ---------------------------------------------------------------- host side
bool code_tc_supported(const Geom& g) {
  return g.N > 0 && (g.S == 3 || g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) && g.Wc >= 8;
}

CodeTcPlan code_tc_plan(const Geom& g, int num_sms) {
  CodeTcPlan p{};
  p.nkg = ceil_div(g.K, 112);
  p.KC = ceil_div(g.K, p.nkg);
  p.Npad = (p.KC + 15) / 16 * 16;
  p.b_bytes = 4 * p.Npad * 128;
  int pitch = g.Wc + g.P;
  while (pitch % 32 != 0) ++pitch;  // lanes are consecutive positions: any pitch is conflict-free within a row
  p.pitch = pitch;
  const int plane = g.Hc * g.Wc;
  p.sw_words = static_cast<size_t>(4 * p.nkg) * plane;
  p.wnc = p.Npad / 4;
  p.wper = 4;
  const int G = num_sms / p.nkg > 0 ? num_sms / p.nkg : 1;
  const int64_t total = static_cast<int64_t>(g.N > 0 ? g.N : 1) * plane;
  int64_t L = total / (8 * static_cast<int64_t>(G));
  L = (L + kCtTile - 1) / kCtTile * kCtTile;
  if (L < kCtTile) L = kCtTile;
  if (L > 4096) L = 4096;
  const int smem_fixed = 1024 + 2 * p.b_bytes;
  auto rows_for = [&](int64_t len) { return static_cast<int>((len + g.Wc - 1) / g.Wc) + 1 + g.P; };
  while (L > kCtTile && smem_fixed + 2 * rows_for(L) * pitch * 4 > kCtSmemMax) L -= kCtTile;
  p.L = static_cast<int>(L);
  p.rs_rows = rows_for(L);
  p.rs_floats = p.rs_rows * pitch;
  p.nseg = ceil_div(plane, p.L);
  p.nitems = g.N * p.nseg;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_fixed + 2 * p.rs_floats * 4;
  p.ok = p.smem <= kCtSmemMax;
  return p;
}

cudaError_t launch_mask_selwords(const Geom& g, const CodeTcPlan& p, uint64_t seed, uint32_t iter, uint64_t thr,
                                 uint32_t* words, cudaStream_t st, int mode, const uint32_t* iter_off) {
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  const int nblk = p.wper * p.nkg;
  const int64_t total = static_cast<int64_t>(nblk) * ((plane + 3) / 4);
  mask_selwords_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(g.K, p.KC, p.wnc, p.wper, nblk,
                                                                                 plane, seed, iter, iter_off, thr, mode,
                                                                                 words);
  return cudaGetLastError();
}

cudaError_t launch_code_tc(const Geom& g, const CodeTcPlan& p, const float* r, const float* d, float* z,
                           const uint32_t* words, const float* tau_dev, float lam, uint32_t* zmax, cudaStream_t st,
                           int tau_stride) {
  CtArgs a{};
  a.r = r; a.d = d; a.z = z; a.mask = words; a.tau = tau_dev; a.lam = lam; a.zmax = zmax;
  a.tau_stride = tau_stride;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.Npad = p.Npad; a.nkg = p.nkg; a.G = p.G;
  a.L = p.L; a.nseg = p.nseg; a.nitems = p.nitems;
  a.pitch = p.pitch; a.rs_rows = p.rs_rows; a.rs_floats = p.rs_floats; a.b_bytes = p.b_bytes;
  switch (g.S) {
    case 3: return run_code_tc_nc<3>(a, p.grid, p.smem, st);
    case 5: return run_code_tc_nc<5>(a, p.grid, p.smem, st);
    case 7: return run_code_tc_nc<7>(a, p.grid, p.smem, st);
    case 9: return run_code_tc_nc<9>(a, p.grid, p.smem, st);
    case 11: return run_code_tc_nc<11>(a, p.grid, p.smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csc

// csc_code_h.cu -- masked proximal-gradient code step, dense-then-mask on the sm_100a tensor cores
// with the 3-term fp16 split (tcgen05.mma kind::f16) and TMA-fed code tiles in the epilogue.
//
// Same step as csc_code_tc.cu (Eq.3-4, §3.1, shrinkage P:311-312, R1/R2):
//   for every masked code (k, u, v) of image n:  c = sum_{a,b} d[k,a,b] r[n,u-P+a,v-P+b],
//   z <- S_{tau lambda}(z - tau c);  unmasked codes are untouched.
// GEMM per 128-position tile: C[p][k] = sum_t R[p][t] d[k][t], M = 128 flattened positions,
// N = Npad filters, K = 128 taps in 8 steps of 16 (kind::f16).  Operands (reading T6):
//   R_s = r * 2^er, d_s = d * 2^ed split as hi = rn11(x_s) (exact fp16), lo = fp16_rn(x_s - hi);
//   C_s = R_hi d_hi + R_hi d_lo + R_lo d_hi (fp32 accumulate), c = C_s * 2^-(er+ed).
//   er comes from max|r| (device scalar written with the residual, csc_api.cu), ed from max|d| over
//   the CTA's filter group (computed in the prologue).
//   A = im2col(r) in TMEM (lane = position, two fp16 taps per 32-bit column), written by the
//       converter warps from the zero-padded residual tile (cp.async, as csc_code_tc.cu).
//   B = the filters, K-major SWIZZLE_128B fp16 (2 K-atoms of 64 taps), resident: 57 KB for 112
//       filters instead of 115 KB for tf32.
// The freed shared memory holds the codes: each epilogue warp owns a {32 positions, NC filters}
// slice and TMA-loads it two tiles ahead (double buffer, own mbarriers), so HBM latency is hidden
// behind two MMA tiles; the warp applies mask / step / shrinkage from shared memory and stores only
// the codes that change (and raises the max|z| bound with them).
// CTA (persistent, 25 warps): warp 0 MMA; warps 1..8 converters; warps 9..24 epilogue.
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kChNS = 4;          // A slots (4 K16-steps = 64 taps each) in TMEM
constexpr int kChConvWarps = 8;
constexpr int kChEpiWarps = 16;
constexpr int kChConvBase = 1, kChEpiBase = kChConvBase + kChConvWarps;
constexpr int kChWarps = kChEpiBase + kChEpiWarps;
constexpr int kChThreads = 32 * kChWarps;
constexpr int kChTile = 128;
constexpr int kChSmemMax = 220 * 1024;

__host__ __device__ constexpr uint32_t idesc_f16_kk(int M, int N) {  // fp16 A/B K-major, fp32 D
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (0u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
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

struct ChArgs {
  const float* r;        // [N][H][W]
  const float* d;        // [K][S][S]
  float* z;              // [N][K][Hc][Wc]
  const uint32_t* mask;  // selection words [nkg*4][plane] or nullptr (all)
  const float* tau;
  const uint32_t* rmax;  // max|r| (float bits)
  uint32_t* zmax;        // raised by every written code, or nullptr
  float lam;
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, nkg, G;
  int L, nseg, nitems;
  int pitch, rs_rows, rs_floats;
  int b_bytes;           // one of hi / lo: 2 K-atoms x Npad rows x 128 B
  int plain;             // 1: z <- c at every position (no z read, no step / shrinkage / mask)
  int tau_stride;        // 0: tau[0] for every filter; 1: tau[k] per filter (ESO rule)
};

struct ChItem {
  int n, p0, p1, ntiles, u_first;
};
__device__ __forceinline__ ChItem ch_item(const ChArgs& A, int item) {
  ChItem it;
  it.n = item / A.nseg;
  const int sg = item - it.n * A.nseg;
  it.p0 = sg * A.L;
  it.p1 = min(it.p0 + A.L, A.Hc * A.Wc);
  it.ntiles = (it.p1 - it.p0 + kChTile - 1) / kChTile;
  it.u_first = it.p0 / A.Wc;
  return it;
}

template <int S, int NC>
__global__ void __launch_bounds__(kChThreads, 1)
code_h_kernel(const __grid_constant__ CUtensorMap tmap_z, const ChArgs A) {
  constexpr int S2 = S * S;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t a_full[kChNS], a_empty[kChNS], acc_full[2], acc_empty[2];
  __shared__ __align__(8) uint64_t z_full[kChEpiWarps][2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t dmax_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  uint8_t* bh = sm;                                        // [2 K-atoms][Npad][128 B] fp16 hi
  uint8_t* bl = sm + A.b_bytes;                            // lo
  float* zsm = reinterpret_cast<float*>(sm + 2 * A.b_bytes);  // [2][16 warps][NC][32] (1 KB aligned)
  float* rs = zsm + 2 * kChEpiWarps * NC * 32;             // [2][rs_rows][pitch]

  // ---- setup: max|d| of this filter group, then the fp16 hi/lo B image (K-major SW128)
  if (tid == 0) dmax_sh = 0u;
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
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kChNS; ++i) {
      mbar_init(&a_full[i], kChConvWarps);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kChEpiWarps);
    }
    for (int w = 0; w < kChEpiWarps; ++w) {
      mbar_init(&z_full[w][0], 1);
      mbar_init(&z_full[w][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  if (warp == kChEpiBase && lane == 0) tma_prefetch_desc(&tmap_z);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  const uint32_t t_acc = tbase;         // 2 x Npad columns
  const uint32_t t_a = tbase + 256u;    // kChNS slots x 64 columns

  if (warp == 0) {
    // ================================ MMA issuer
    const uint32_t idesc = idesc_f16_kk(128, A.Npad);
    const uint32_t sbh = su32(bh), sbl = su32(bl);
    const uint32_t katom = static_cast<uint32_t>(A.Npad) * 128u;
    uint32_t g = 0, tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const ChItem it = ch_item(A, item);
      for (int tl = 0; tl < it.ntiles; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_after();
        const uint32_t dcol = t_acc + buf * static_cast<uint32_t>(A.Npad);
        for (int j = 0; j < 2; ++j, ++g) {  // 2 slots of 4 K16-steps (64 taps)
          const uint32_t slot = g % kChNS, ph = (g / kChNS) & 1u;
          mbar_wait(&a_full[slot], ph);
          tc_after();
          const uint32_t ah = t_a + slot * 64u;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // K16-step 4j + e: K-atom j, 32 B (16 fp16) into the 128-B row
            const uint64_t dbh = sdesc(sbh + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint64_t dbl = sdesc(sbl + j * katom + 32u * e, 16u, 1024u, kLayout128B);
            const uint32_t acc0 = (j > 0 || e > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred e, p, t;\n"
                "elect.sync _|e, 0xffffffff;\n"
                "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %4, p;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %6, %4, t;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %4, t;\n"
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
  } else if (warp < kChEpiBase) {
    // ================================ converters: im2col(r) -> TMEM, two fp16 taps per column
    const int cw = warp - kChConvBase;  // 0..7
    const int q = warp & 3;
    const int h = cw >> 2;              // K16-steps {2h, 2h+1} of every slot
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const int ct = tid - 32 * kChConvBase;
    const float sr = exp2i_h(er);
    auto stage_r = [&](int item, int buf) {
      const ChItem it = ch_item(A, item);
      float* dst = rs + buf * A.rs_floats;
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      for (int e = ct; e < A.rs_floats; e += 32 * kChConvWarps) {
        const int rho = e / A.pitch, c = e - rho * A.pitch;
        const int i = it.u_first - A.P + rho, jj = c - A.P;
        const bool ok = i >= 0 && i < A.H && jj >= 0 && jj < A.W;
        cp_async4(su32(dst + e), ok ? rn + static_cast<size_t>(i) * A.W + jj : rn, ok);
      }
      cp_async_commit();
    };
    auto body = [&](auto hc) {
      constexpr int H = decltype(hc)::value;
      uint32_t g = 0;
      int ibuf = 0;
      if (gi < A.nitems) stage_r(gi, 0);
      for (int item = gi; item < A.nitems; item += A.G, ibuf ^= 1) {
        const ChItem it = ch_item(A, item);
        if (item + A.G < A.nitems) stage_r(item + A.G, ibuf ^ 1);
        else cp_async_commit();
        cp_async_wait<1>();
        named_sync(1, 32 * kChConvWarps);
        const float* rtile = rs + ibuf * A.rs_floats;
        for (int tl = 0; tl < it.ntiles; ++tl) {
          const int p = it.p0 + tl * kChTile + 32 * q + lane;
          const bool pok = p < it.p1;
          const int u = p / A.Wc, v = p - u * A.Wc;
          const float* src = rtile + (pok ? (u - it.u_first) * A.pitch + v : 0);
#pragma unroll
          for (int j = 0; j < 2; ++j, ++g) {  // slot j: taps 64 j .. 64 j + 63
            const uint32_t slot = g % kChNS, ph = (g / kChNS) & 1u;
            mbar_wait_sleep(&a_empty[slot], ph ^ 1u);
            tc_after();
#pragma unroll
            for (int ee = 0; ee < 2; ++ee) {
              const int e = 2 * H + ee;  // K16-step within the slot
              uint32_t hv[8], lv[8];
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const int t0 = 64 * j + 16 * e + 2 * jj, t1 = t0 + 1;
                const float x0 = (t0 < S2 && pok) ? src[(t0 / S) * A.pitch + (t0 % S)] * sr : 0.f;
                const float x1 = (t1 < S2 && pok) ? src[(t1 / S) * A.pitch + (t1 % S)] * sr : 0.f;
                const float h0 = rn11_h(x0), h1 = rn11_h(x1);
                hv[jj] = pack_h2_h(h0, h1);
                lv[jj] = pack_h2_h(x0 - h0, x1 - h1);
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
        named_sync(1, 32 * kChConvWarps);
      }
    };
    if (h == 0) body(std::integral_constant<int, 0>{});
    else body(std::integral_constant<int, 1>{});
    cp_async_wait<0>();
  } else {
    // ================================ epilogue: z <- S(z - tau c) on masked codes
    const int ew = warp - kChEpiBase;  // 0..15
    const int q = warp & 3;
    const int cb = ew >> 2;            // filter block of NC
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const bool plain = A.plain != 0;
    const float tau = plain ? 0.f : *A.tau;
    const float kappa = tau * A.lam;
    const float inv = exp2i_h(-(er + ed));
    const size_t plane = static_cast<size_t>(A.Hc) * A.Wc;
    const int k0 = kg * A.KC + cb * NC;
    const int kend = min(kg * A.KC + A.KC, A.K);
    float* zs0 = zsm + ew * NC * 32;                 // buffer b at zs0 + b * kChEpiWarps * NC * 32
    const uint32_t zbytes = static_cast<uint32_t>(NC) * 128u;
    // the sequence of (item, tile) this warp consumes, advanced by one per step
    auto advance = [&](int& item, int& tl) {
      const ChItem it = ch_item(A, item);
      if (++tl >= it.ntiles) {
        tl = 0;
        item += A.G;
      }
    };
    auto issue = [&](int item, int tl, int b) {  // TMA {32 positions, NC planes} of tile (item, tl)
      if (plain || item >= A.nitems || lane != 0) return;
      const ChItem it = ch_item(A, item);
      const int pw = it.p0 + tl * kChTile + 32 * q;
      mbar_arrive_expect_tx(&z_full[ew][b], zbytes);
      tma_load_2d(su32(zs0 + b * kChEpiWarps * NC * 32), &tmap_z, pw, it.n * A.K + k0, &z_full[ew][b]);
    };
    float wmax = 0.f;
    int item = gi, tl = 0;
    int pi = gi, ptl = 0;  // prefetch cursor: two tiles ahead
    issue(pi, ptl, 0);
    if (pi < A.nitems) advance(pi, ptl);
    issue(pi, ptl, 1);
    if (pi < A.nitems) advance(pi, ptl);
    uint32_t tcount = 0;
    while (item < A.nitems) {
      const ChItem it = ch_item(A, item);
      const uint32_t buf = tcount & 1u, use = tcount >> 1;
      const int pw = it.p0 + tl * kChTile + 32 * q;
      const int p = pw + lane;
      const bool pok = p < it.p1;
      const int nvk = kend - k0;  // filters of this warp's block that exist (the rest is padding)
      const uint32_t kbits = nvk >= 32 ? 0xffffffffu : (nvk <= 0 ? 0u : ((1u << nvk) - 1u));
      const uint32_t sel = kbits & (A.mask == nullptr ? (pok ? 0xffffffffu : 0u)
                                                      : (pok ? __ldg(A.mask + static_cast<size_t>(kg * 4 + cb) * plane + p) : 0u));
      float* zb = A.z + (static_cast<size_t>(it.n) * A.K + k0) * plane + p;
      const float* zs = zs0 + buf * kChEpiWarps * NC * 32;
      if (!plain) mbar_wait_sleep(&z_full[ew][buf], use & 1u);
      mbar_wait_sleep(&acc_full[buf], use & 1u);
      tc_after();
      const uint32_t colb = t_acc + buf * static_cast<uint32_t>(A.Npad) + static_cast<uint32_t>(cb * NC);
      // per-filter step sizes (ESO rule) in a separate instantiation of the loop, so the
      // scalar-tau hot path carries no extra loads
      const float ntinv = -tau * inv;
      auto epi = [&](auto per_k) {
        constexpr bool PK = decltype(per_k)::value;
#pragma unroll
        for (int j4 = 0; j4 < NC / 4; ++j4) {
          float c4[4];
          tmem_ld4_nowait(tq + colb + 4u * j4, c4);
          tmem_ld_wait();
          if (plain) {
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const int i = 4 * j4 + i4;
              if (pok && (k0 + i) < kend) zb[static_cast<size_t>(i) * plane] = c4[i4] * inv;
            }
            continue;
          }
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            const int i = 4 * j4 + i4;
            const float zv = zs[i * 32 + lane];
            const float tk = PK ? __ldg(A.tau + min(k0 + i, A.K - 1)) : tau;
            const float kk = PK ? tk * A.lam : kappa;
            // -tau * (c * 2^-(er+ed)) with one multiply: scaling by a power of two is exact
            const float w = fmaf(PK ? -tk * inv : ntinv, c4[i4], zv);
            const float nz = w - fminf(fmaxf(w, -kk), kk);  // S_kk(w): w -/+ kk outside [-kk, kk], +0 inside
            if (((sel >> i) & 1u) && nz != zv) {
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
      fence_async_shared();  // generic reads of the slice before the async-proxy refill
      __syncwarp();
      issue(pi, ptl, static_cast<int>(buf));
      if (pi < A.nitems) advance(pi, ptl);
      advance(item, tl);
      ++tcount;
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

typedef CUresult (*PFN_encodeTiled_ch)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_ch encode_fn_ch() {
  static PFN_encodeTiled_ch fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_ch>(p);
  }
  return fn;
}

template <int S, int NC>
cudaError_t run_code_h(const CUtensorMap& tm, const ChArgs& a, int grid, int smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(code_h_kernel<S, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, kChSmemMax);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  code_h_kernel<S, NC><<<grid, kChThreads, smem, st>>>(tm, a);
  return cudaGetLastError();
}

template <int S>
cudaError_t run_code_h_nc(const CUtensorMap& tm, const ChArgs& a, int grid, int smem, cudaStream_t st) {
  switch (a.Npad / 4) {
    case 4: return run_code_h<S, 4>(tm, a, grid, smem, st);
    case 8: return run_code_h<S, 8>(tm, a, grid, smem, st);
    case 12: return run_code_h<S, 12>(tm, a, grid, smem, st);
    case 16: return run_code_h<S, 16>(tm, a, grid, smem, st);
    case 20: return run_code_h<S, 20>(tm, a, grid, smem, st);
    case 24: return run_code_h<S, 24>(tm, a, grid, smem, st);
    case 28: return run_code_h<S, 28>(tm, a, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// ---------------------------------------------------------------- host side
bool code_h_supported(const Geom& g) {
  return g.N > 0 && (g.S == 3 || g.S == 5 || g.S == 7 || g.S == 9 || g.S == 11) && g.Wc >= 8 &&
         (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 && encode_fn_ch() != nullptr;
}

CodeTcPlan code_h_plan(const Geom& g, int num_sms) {
  CodeTcPlan p{};
  p.nkg = ceil_div(g.K, 112);
  p.KC = ceil_div(g.K, p.nkg);
  p.Npad = (p.KC + 15) / 16 * 16;
  p.b_bytes = 2 * p.Npad * 128;
  int pitch = g.Wc + g.P;
  while (pitch % 32 != 0) ++pitch;
  p.pitch = pitch;
  const int plane = g.Hc * g.Wc;
  p.sw_words = static_cast<size_t>(4 * p.nkg) * plane;
  const int G = num_sms / p.nkg > 0 ? num_sms / p.nkg : 1;
  const int64_t total = static_cast<int64_t>(g.N > 0 ? g.N : 1) * plane;
  int64_t L = total / (8 * static_cast<int64_t>(G));
  L = (L + kChTile - 1) / kChTile * kChTile;
  if (L < kChTile) L = kChTile;
  if (L > 4096) L = 4096;
  const int zbytes = 2 * kChEpiWarps * (p.Npad / 4) * 32 * 4;
  const int smem_fixed = 1024 + 2 * p.b_bytes + zbytes;
  auto rows_for = [&](int64_t len) { return static_cast<int>((len + g.Wc - 1) / g.Wc) + 1 + g.P; };
  while (L > kChTile && smem_fixed + 2 * rows_for(L) * pitch * 4 > kChSmemMax) L -= kChTile;
  p.L = static_cast<int>(L);
  p.rs_rows = rows_for(L);
  p.rs_floats = p.rs_rows * pitch;
  p.nseg = ceil_div(plane, p.L);
  p.nitems = g.N * p.nseg;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_fixed + 2 * p.rs_floats * 4;
  p.ok = p.smem <= kChSmemMax;
  p.half = true;
  return p;
}

cudaError_t launch_code_h(const Geom& g, const CodeTcPlan& p, const float* r, const float* d, float* z,
                          const uint32_t* words, const float* tau_dev, float lam, const uint32_t* rmax,
                          uint32_t* zmax, cudaStream_t st, bool plain, int tau_stride) {
  static const float* cached_z = nullptr;
  static Geom cached_g{};
  static int cached_nc = 0;
  static CUtensorMap tm;
  const int NC = p.Npad / 4;
  if (z != cached_z || std::memcmp(&cached_g, &g, sizeof(Geom)) != 0 || cached_nc != NC) {
    PFN_encodeTiled_ch enc = encode_fn_ch();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.Hc) * g.Wc, static_cast<cuuint64_t>(g.N) * g.K};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.Hc) * g.Wc * 4};
    const cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(NC)};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, z, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidPitchValue;
    cached_z = z;
    cached_g = g;
    cached_nc = NC;
  }
  ChArgs a{};
  a.r = r; a.d = d; a.z = z; a.mask = words; a.tau = tau_dev; a.lam = lam; a.rmax = rmax; a.zmax = zmax;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.Npad = p.Npad; a.nkg = p.nkg; a.G = p.G;
  a.L = p.L; a.nseg = p.nseg; a.nitems = p.nitems;
  a.pitch = p.pitch; a.rs_rows = p.rs_rows; a.rs_floats = p.rs_floats; a.b_bytes = p.b_bytes;
  a.plain = plain ? 1 : 0;
  a.tau_stride = tau_stride;
  if (plain) {
    a.mask = nullptr;
    a.zmax = nullptr;
  }
  switch (g.S) {
    case 3: return run_code_h_nc<3>(tm, a, p.grid, p.smem, st);
    case 5: return run_code_h_nc<5>(tm, a, p.grid, p.smem, st);
    case 7: return run_code_h_nc<7>(tm, a, p.grid, p.smem, st);
    case 9: return run_code_h_nc<9>(tm, a, p.grid, p.smem, st);
    case 11: return run_code_h_nc<11>(tm, a, p.grid, p.smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csc

// csc_wgrad_tc.cu -- filter gradient g = Z^T r on the sm_100a tensor cores (tcgen05, 3xTF32).
//
// Gradient of the Eq.5 fit term (§3.1): for every filter k and tap t = (a, b)
//   g[k][t] = sum_n sum_{(u,v)} z[n,k,u,v] * R_n[(u,v)][t],   R_n[(u,v)][(a,b)] = r[n, u-P+a, v-P+b]
// (r = 0 outside the H x W image), i.e. the correlation of the residual with every code map.
// As a GEMM per CTA:   D[t][k] += sum_pos A[t][pos] * B[k][pos]
//   M = 128 taps (s^2 <= 121 used), N = Npad filters of one k-group, K = code positions,
//   8 positions per tcgen05.mma (kind::tf32), 3 products per K-step (3xTF32:
//   A_hi B_hi + A_hi B_lo + A_lo B_hi, hi = the fp32 value read as tf32, lo = x - trunc_tf32(x)).
// Operands:
//   B = z, straight from HBM by TMA: box {32 flattened positions, KC filter planes}, SWIZZLE_128B,
//       which is the canonical K-major SW128 UMMA layout (row = filter, 128 B = 32 positions).
//       The converter warps add the lo copy of each stage in shared memory.
//   A = im2col of r, built by the converter warps in TMEM (lane = tap, column = position):
//       each lane reads 8 consecutive positions of its shifted residual row from a zero-padded
//       shared-memory tile (pitch = s mod 32, so the 32 taps of a warp hit 32 banks).
// Positions run row by row over (u, v < Wc8 = roundup8(Wc)); the columns v >= Wc read only the
// zero padding of the residual tile, so the z values TMA brings for them (the next row's codes)
// are multiplied by 0.  The accumulator restarts every tile (<= 8 chunks of 32 positions of one
// code row) and the epilogue warps add it into fp64 registers, so fp32 accumulation never spans
// more than 96 tensor-core accumulation steps; the per-CTA fp64 partials are summed over CTAs in
// a fixed order by wgrad_reduce_kernel (deterministic).
//
// CTA (persistent, one per SM, 26 warps):
//   warp 0       MMA issue (one elected lane)          warp 1       TMA producer (one lane)
//   warps 2..9   converters: z lo copy + r im2col -> TMEM A slots, residual tile staging (cp.async)
//   warps 10..25 epilogue: TMEM accumulator -> fp64 registers (4 warps per TMEM lane quarter)
#include "csc_internal.cuh"
#include "csc_tc_ptx.cuh"

#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

namespace csc {
namespace {

using namespace tcx;

constexpr int kWgNS = 4;          // pipeline stages (z stage in smem + A slot in TMEM)
constexpr int kWgConvWarps = 8;   // converter warps (2 per TMEM lane quarter)
constexpr int kWgEpiWarps = 16;   // epilogue warps (4 per lane quarter)
constexpr int kWgConvBase = 2, kWgEpiBase = kWgConvBase + kWgConvWarps;
constexpr int kWgWarps = kWgEpiBase + kWgEpiWarps;
constexpr int kWgThreadsTc = 32 * kWgWarps;
constexpr int kWgFlush = 32;     // accumulator tiles summed in fp32 before each fp64 flush (epilogue)
constexpr int kWgMaxCpt = 2;      // chunks (32 positions) per accumulator tile (default; CSC_WG_CPT overrides)
constexpr int kWgSmemMax = 220 * 1024;

struct WgArgs {
  const float* r;      // [N][H][W]
  double* gpart;       // [G][K][S*S]
  int N, K, S, H, W, Hc, Wc, P;
  int KC, Npad, nkg, G;
  int L, nseg, nitems;   // item = (image, segment of L flattened positions, L % 32 == 0)
  int pitch, rs_rows, rs_floats;  // residual tile
  int stage_bytes;       // one of hi / lo
  int cpt;               // chunks (32 positions) per accumulator tile
  unsigned long long* tdbg;  // CSC_WG_TIMING: per-CTA role timings [grid][8] or nullptr
  int dbg;  // CSC_WG_DEBUG development switches: 1 no MMA, 2 no TMA, 4 no tmem st, 8 no tmem ld, 16 no lo copy
};

// Item = (image n, flattened code positions [p0, p1) of the plane, p0 % 32 == 0).
struct WgItem {
  int n, p0, p1, nch, u_first;
};
__device__ __forceinline__ WgItem wg_item(const WgArgs& A, int item) {
  WgItem it;
  it.n = item / A.nseg;
  const int sg = item - it.n * A.nseg;
  const int plane = A.Hc * A.Wc;
  it.p0 = sg * A.L;
  it.p1 = min(it.p0 + A.L, plane);
  it.nch = (it.p1 - it.p0 + 31) >> 5;
  it.u_first = it.p0 / A.Wc;
  return it;
}
__device__ __forceinline__ int wg_ntiles(int nch, int cpt) { return (nch + cpt - 1) / cpt; }

template <int NC>
__global__ void __launch_bounds__(kWgThreadsTc, 1)
wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmap_z, const WgArgs A) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t z_full[kWgNS], ready[kWgNS], empty[kWgNS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = __shfl_sync(kFullMask, tid >> 5, 0), lane = tid & 31;
  const int gi = blockIdx.x % A.G, kg = blockIdx.x / A.G;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  uint8_t* stages = sm;                                   // [NS][hi | lo], each stage_bytes
  float* rs = reinterpret_cast<float*>(sm + 2 * kWgNS * A.stage_bytes);  // [2][rs_rows][pitch]: r, then hi
  float* rsl = rs + 2 * A.rs_floats;                                      // [2][rs_rows][pitch]: lo

  // ---- setup: zero the z stages (rows >= KC are never written by TMA), barriers, TMEM
  for (int e = tid; e < 2 * kWgNS * A.stage_bytes / 16; e += kWgThreadsTc)
    reinterpret_cast<int4*>(stages)[e] = make_int4(0, 0, 0, 0);
  fence_async_shared();
  if (tid == 0) {
    for (int i = 0; i < kWgNS; ++i) {
      mbar_init(&z_full[i], 1);
      mbar_init(&ready[i], 4);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kWgEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 1 && lane == 0) tma_prefetch_desc(&tmap_z);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = __shfl_sync(kFullMask, tmem_base_sh, 0);
  const uint32_t t_acc = tbase;          // 2 x Npad columns
  const uint32_t t_a = tbase + 256u;     // NS slots x 64 columns (4 K-steps x (8 hi + 8 lo))

  if (warp == 0) {
    // ================================ MMA issuer
    const uint32_t idesc = idesc_tf32(128, A.Npad, 0, 0);
    unsigned long long w_acc = 0, w_rdy = 0;
    const unsigned long long t_beg = clock64();
    uint32_t g = 0, tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WgItem it = wg_item(A, item);
      const int ntl = wg_ntiles(it.nch, A.cpt);
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        const unsigned long long tw0 = clock64();
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        w_acc += clock64() - tw0;
        tc_after();
        const uint32_t d = t_acc + buf * static_cast<uint32_t>(A.Npad);
        const int c0 = tl * A.cpt, c1 = min(c0 + A.cpt, it.nch);
        for (int c = c0; c < c1; ++c, ++g) {
          const uint32_t slot = g % kWgNS, ph = (g / kWgNS) & 1u;
          const unsigned long long tw1 = clock64();
          mbar_wait(&ready[slot], ph);
          w_rdy += clock64() - tw1;
          tc_after();
          const int nks = min(4, (it.p1 - it.p0 - 32 * c + 7) >> 3);
          const uint32_t sh = su32(stages + slot * 2 * A.stage_bytes);
          const uint32_t sl = sh + A.stage_bytes;
          const uint32_t ah = t_a + slot * 64u;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e < nks && !(A.dbg & 1)) {
              const uint64_t bh = sdesc(sh + 32u * e, 16u, 1024u, kLayout128B);
              const uint64_t bl = sdesc(sl + 32u * e, 16u, 1024u, kLayout128B);
              const uint32_t acc0 = (c > c0 || e > 0) ? 1u : 0u;
              asm volatile(
                  "{\n.reg .pred e, p, t;\n"
                  "elect.sync _|e, 0xffffffff;\n"
                  "setp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 1, 1;\n"
                  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, p;\n"
                  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %4, t;\n"
                  "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %4, t;\n"
                  "}\n" ::"r"(d),
                  "r"(ah + 8u * e), "r"(ah + 32u + 8u * e), "l"(bh), "r"(idesc), "r"(acc0), "l"(bl)
                  : "memory");
            }
          }
          mma_commit_elect(&empty[slot]);
        }
        mma_commit_elect(&acc_full[buf]);
      }
    }
    if (A.tdbg != nullptr && lane == 0) {
      A.tdbg[blockIdx.x * 8 + 0] = clock64() - t_beg;
      A.tdbg[blockIdx.x * 8 + 1] = w_acc;
      A.tdbg[blockIdx.x * 8 + 2] = w_rdy;
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================ TMA producer
    if (lane == 0) {
      const uint32_t bytes = 32u * 4u * static_cast<uint32_t>(A.KC);
      const int plane0 = kg * A.KC;
      uint32_t g = 0;
      for (int item = gi; item < A.nitems; item += A.G) {
        const WgItem it = wg_item(A, item);
        for (int c = 0; c < it.nch; ++c, ++g) {
          const uint32_t slot = g % kWgNS, ph = (g / kWgNS) & 1u;
          mbar_wait(&empty[slot], ph ^ 1u);
          if (A.dbg & 2) {
            mbar_arrive(&z_full[slot]);
            continue;
          }
          mbar_arrive_expect_tx(&z_full[slot], bytes);
          // inner coordinate it.p0 + 32c is a multiple of 32 floats: TMA needs 16-B aligned box starts
          tma_load_2d(su32(stages + slot * 2 * A.stage_bytes), &tmap_z, it.p0 + 32 * c, it.n * A.K + plane0,
                      &z_full[slot]);
        }
      }
    }
    __syncwarp();
  } else if (warp < kWgEpiBase) {
    // ================================ converters
    const int cw = warp - kWgConvBase;  // 0..7
    const int q = warp & 3;             // TMEM lane quarter
    const int grp = cw >> 2;            // the two groups of 4 warps take alternate chunks (whole chunks),
                                        // so two chunks are converted concurrently
    const int ctg = (cw & 3) * 32 + lane;  // 0..127 within the group
    const int t = 32 * q + lane;        // tap of this lane
    const int S2 = A.S * A.S;
    const bool tap_ok = t < S2;
    const int ta = tap_ok ? t / A.S : 0, tb = tap_ok ? t - ta * A.S : 0;
    const int tap_off = ta * A.pitch + tb;
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    const int ct = tid - 32 * kWgConvBase;  // 0..255
    // residual tile staging for one item: rs[rho][c] = r[n, u_first-P+rho, c-P] (0 outside)
    auto stage_r = [&](int item, int buf) {
      const WgItem it = wg_item(A, item);
      float* dst = rs + buf * A.rs_floats;
      const float* rn = A.r + static_cast<size_t>(it.n) * A.H * A.W;
      for (int e = ct; e < A.rs_floats; e += 32 * kWgConvWarps) {
        const int rho = e / A.pitch, c = e - rho * A.pitch;
        const int i = it.u_first - A.P + rho, j = c - A.P;
        const bool ok = i >= 0 && i < A.H && j >= 0 && j < A.W;
        cp_async4(su32(dst + e), ok ? rn + static_cast<size_t>(i) * A.W + j : rn, ok);
      }
      cp_async_commit();
    };
    uint32_t g = 0;
    unsigned long long w_zf = 0, w_lo = 0, w_im = 0, w_st = 0;
    const unsigned long long t_cv = clock64();
    int ibuf = 0;
    if (gi < A.nitems) stage_r(gi, 0);
    for (int item = gi; item < A.nitems; item += A.G, ibuf ^= 1) {
      const WgItem it = wg_item(A, item);
      if (item + A.G < A.nitems) stage_r(item + A.G, ibuf ^ 1);
      else cp_async_commit();
      cp_async_wait<1>();
      named_sync(1, 32 * kWgConvWarps);
      // split the staged residual tile once (hi in place, lo beside it): the im2col below reads
      // every value once per tap, so this removes ~121 redundant splits per value
      {
        float* th = rs + ibuf * A.rs_floats;
        float* tl = rsl + ibuf * A.rs_floats;
        for (int e = ct; e < A.rs_floats; e += 32 * kWgConvWarps) {
          float hf, lf;
          tf32_split_rn(th[e], hf, lf);
          th[e] = hf;
          tl[e] = lf;
        }
      }
      named_sync(1, 32 * kWgConvWarps);
      const float* rtile = rs + ibuf * A.rs_floats + tap_off;
      const float* rtilel = rsl + ibuf * A.rs_floats + tap_off;
      for (int c = 0; c < it.nch; ++c, ++g) {
        if (static_cast<int>(g & 1u) != grp) continue;
        const uint32_t slot = g % kWgNS, ph = (g / kWgNS) & 1u;
        // first position of the chunk, as (row, column) -- warp-uniform
        const int pk = it.p0 + 32 * c;
        int u = pk / A.Wc;
        int v = pk - u * A.Wc;
        const unsigned long long tw2 = clock64();
        mbar_wait_sleep(&z_full[slot], ph);
        w_zf += clock64() - tw2;
        const unsigned long long tl0 = clock64();
        // (1) lo copy of the z stage (elementwise, the swizzle is irrelevant)
        if (!(A.dbg & 16)) {
          float4* hi4 = reinterpret_cast<float4*>(stages + slot * 2 * A.stage_bytes);
          float4* lo4 = reinterpret_cast<float4*>(stages + slot * 2 * A.stage_bytes + A.stage_bytes);
          const int n4 = A.KC * 8;  // KC rows x 32 floats / 4
          // hi stays the fp32 z in place (the tensor core reads its tf32 truncation); lo = z - trunc(z)
          // exactly, itself truncated to tf32 by the tensor core (reading T1'')
          for (int e = ctg; e < n4; e += 128) {
            const float4 x = hi4[e];
            float4 l;
            l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
            l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
            l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
            l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
            lo4[e] = l;
          }
        }
        const unsigned long long tl1 = clock64();
        w_lo += tl1 - tl0;
        // (2) im2col of r into the A slot: the 4 K-steps of this chunk for this lane quarter.
        // R[(u,v)][(a,b)] = r[u-P+a][v-P+b] = rs[u - u_first + a][v + b]
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int p = pk + 8 * e;  // first position of K-step e
          if (p < it.p1) {
            uint32_t hv[8], lv[8];
            if (v + 7 < A.Wc && p + 7 < it.p1) {
              const int o = (u - it.u_first) * A.pitch + v;
              const float* srch = rtile + o;
              const float* srcl = rtilel + o;
              // lanes of taps t >= s^2 load the tile at tap offset 0: their accumulator rows are never
              // read (the epilogue stores t < s^2 only), and D row t depends on A row t alone
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                hv[j] = __float_as_uint(srch[j]);
                lv[j] = __float_as_uint(srcl[j]);
              }
            } else {
              // row wrap (Wc >= 8: at most one) or end of the item
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int vj = v + j;
                const bool wrap = vj >= A.Wc;
                const int uu = wrap ? u + 1 : u, vv = wrap ? vj - A.Wc : vj;
                const bool ok = p + j < it.p1;
                const int o = (uu - it.u_first) * A.pitch + vv;
                hv[j] = ok ? __float_as_uint(rtile[o]) : 0u;
                lv[j] = ok ? __float_as_uint(rtilel[o]) : 0u;
              }
            }
            const uint32_t ta_col = t_a + slot * 64u + 8u * e;
            if (!(A.dbg & 4)) {
              tmem_st8(tq + ta_col, hv);
              tmem_st8(tq + ta_col + 32u, lv);
            }
          }
          v += 8;
          if (v >= A.Wc) {
            v -= A.Wc;
            ++u;
          }
        }
        const unsigned long long tl2 = clock64();
        w_im += tl2 - tl1;
        fence_async_shared();
        tmem_st_wait();
        tc_before();
        __syncwarp();
        w_st += clock64() - tl2;
        if (lane == 0) mbar_arrive(&ready[slot]);
      }
      named_sync(1, 32 * kWgConvWarps);  // everyone is done reading rs[ibuf] before it is restaged
    }
    cp_async_wait<0>();
    if (A.tdbg != nullptr && warp == kWgConvBase && lane == 0) {
      A.tdbg[blockIdx.x * 8 + 3] = w_zf;
      A.tdbg[blockIdx.x * 8 + 4] = clock64() - t_cv;
      A.tdbg[blockIdx.x * 8 + 5] = w_lo;
      A.tdbg[blockIdx.x * 8 + 6] = w_im;
      A.tdbg[blockIdx.x * 8 + 7] = w_st;
    }
  } else {
    // ================================ epilogue
    const int ew = warp - kWgEpiBase;  // 0..15
    const int q = warp & 3;
    const int cb = ew >> 2;            // column block (NC columns)
    // the tile sums (fp32 from TMEM) accumulate in plain fp32 registers over kWgFlush tiles (round to
    // nearest: an unbiased error of ~sqrt(kWgFlush) 2^-24 of the block sum), and each block sum is added
    // into the CTA's fp64 partial gpart[gi] in global memory (L2-resident, this CTA's own rows): NC live
    // accumulators instead of a 2 NC-register compensated state (which spilled at 72 registers)
    const int t = 32 * q + lane;
    const int S2 = A.S * A.S;
    float acc[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = 0.f;
    int nacc = 0;
    bool first = true;
    double* const gp0 = A.gpart + (static_cast<size_t>(gi) * A.K + kg * A.KC + cb * NC) * S2 + t;
    const int nvalid = min(NC, min(A.KC - cb * NC, A.K - kg * A.KC - cb * NC));  // real filters of the block
    auto flush = [&]() {
      if (t < S2) {
        // the first block is stored, later ones are added with fire-and-forget fp64 reductions; one thread
        // owns each element, and same-address operations of a thread keep program order: deterministic
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          if (i < nvalid) {
            double* gp = gp0 + static_cast<size_t>(i) * S2;
            if (first) *gp = static_cast<double>(acc[i]);
            else atomicAdd(gp, static_cast<double>(acc[i]));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) acc[i] = 0.f;
      first = false;
      nacc = 0;
    };
    const uint32_t tq = (static_cast<uint32_t>(32 * q) << 16);
    uint32_t tcount = 0;
    for (int item = gi; item < A.nitems; item += A.G) {
      const WgItem it = wg_item(A, item);
      const int ntl = wg_ntiles(it.nch, A.cpt);
      for (int tl = 0; tl < ntl; ++tl, ++tcount) {
        const uint32_t buf = tcount & 1u, use = tcount >> 1;
        mbar_wait_sleep(&acc_full[buf], use & 1u);
        tc_after();
        const uint32_t col = t_acc + buf * static_cast<uint32_t>(A.Npad) + static_cast<uint32_t>(cb * NC);
        float f[NC];
#pragma unroll
        for (int j = 0; j < NC / 4; ++j) tmem_ld4_nowait(tq + col + 4u * j, *reinterpret_cast<float(*)[4]>(f + 4 * j));
        tmem_ld_wait();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
#pragma unroll
        for (int i = 0; i < NC / 2; ++i) {
          const float2 a2 = __fadd2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), make_float2(f[2 * i], f[2 * i + 1]));
          acc[2 * i] = a2.x;
          acc[2 * i + 1] = a2.y;
        }
        const bool last = tl + 1 == ntl && item + A.G >= A.nitems;
        if (++nacc == kWgFlush || last) flush();
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
cudaError_t run_wgrad_tc(const CUtensorMap& tm, const WgArgs& a, int grid, int smem, cudaStream_t st) {
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(&wgrad_tc_kernel<NC>), kWgSmemMax);
  if (e != cudaSuccess) return e;
#ifdef CSC_ROLE_TIMING
  static unsigned long long* dbg = nullptr;
  static int calls = 0;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 8 * 1024);
  cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 8 * 1024, st);
  WgArgs b = a;
  b.tdbg = dbg;
  wgrad_tc_kernel<NC><<<grid, kWgThreadsTc, smem, st>>>(tm, b);
  if (++calls % 4 == 0) {
    static unsigned long long h[8 * 1024];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost);
    double t[8] = {0};
    for (int bk = 0; bk < grid; ++bk)
      for (int i = 0; i < 8; ++i) t[i] += static_cast<double>(h[bk * 8 + i]) / grid;
    fprintf(stderr,
            "[wgrad roles] mma: total %.0f w_accempty %.0f w_ready %.0f | conv0: w_z %.0f total %.0f lo %.0f im2col %.0f "
            "stwait %.0f\n",
            t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
  }
#else
  wgrad_tc_kernel<NC><<<grid, kWgThreadsTc, smem, st>>>(tm, a);
#endif
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- host side
bool wgrad_tc_supported(const Geom& g) {
  return g.N > 0 && g.S >= 3 && g.S * g.S <= 128 && g.Wc >= 8 && (static_cast<int64_t>(g.Hc) * g.Wc) % 4 == 0 &&
         static_cast<int64_t>(g.N) * g.K < (int64_t(1) << 31) && tmap_available();
}

WgTcPlan wgrad_tc_plan(const Geom& g, int num_sms) {
  WgTcPlan p{};
  // filters per k-group: <= 112 so that the epilogue's fp64 accumulators fit (NC <= 28)
  p.nkg = ceil_div(g.K, 112);
  p.KC = ceil_div(g.K, p.nkg);
  p.Npad = (p.KC + 15) / 16 * 16;
  p.stage_bytes = p.Npad * 128;
  // residual tile pitch: >= Wc + P, == S (mod 32) so that the 32 taps of a lane quarter hit 32 banks
  int pitch = g.Wc + g.P;
  while (pitch % 32 != g.S % 32) ++pitch;
  p.pitch = pitch;
  // items: (image, segment of L positions); ~>= 12 items per CTA, L a multiple of 32
  const int plane = g.Hc * g.Wc;
  const int G = num_sms / p.nkg > 0 ? num_sms / p.nkg : 1;
  const int64_t total = static_cast<int64_t>(g.N > 0 ? g.N : 1) * plane;
  int64_t L = total / (12 * static_cast<int64_t>(G));
  L = (L + 31) / 32 * 32;
  if (L < 256) L = 256;
  if (L > 4096) L = 4096;
  const int smem_fixed = 1024 + 2 * kWgNS * p.stage_bytes;
  auto rows_for = [&](int64_t len) { return static_cast<int>((len + g.Wc - 1) / g.Wc) + 1 + g.P; };
  while (L > 32 && smem_fixed + 4 * rows_for(L) * pitch * 4 > kWgSmemMax) L -= 32;
  p.L = static_cast<int>(L);
  p.rs_rows = rows_for(L);
  p.rs_floats = p.rs_rows * pitch;
  p.nseg = ceil_div(plane, p.L);
  p.nitems = g.N * p.nseg;
  p.G = p.nitems < G ? (p.nitems > 0 ? p.nitems : 1) : G;
  p.grid = p.G * p.nkg;
  p.smem = smem_fixed + 4 * p.rs_floats * 4;
  return p;
}

cudaError_t launch_wgrad_tc(const Geom& g, const WgTcPlan& p, TmapCache* tmc, const float* z, const float* r,
                            double* gpart, cudaStream_t st) {
  const uint64_t plane = static_cast<uint64_t>(g.Hc) * g.Wc;
  cudaError_t e0 = tmap_2d(*tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, plane, static_cast<uint64_t>(g.N) * g.K, plane * 4,
                           32, static_cast<uint32_t>(p.KC), CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (e0 != cudaSuccess) return e0;
  const CUtensorMap& tm = tmc->map;
  WgArgs a{};
  a.r = r;
  a.gpart = gpart;
  a.N = g.N; a.K = g.K; a.S = g.S; a.H = g.H; a.W = g.W; a.Hc = g.Hc; a.Wc = g.Wc; a.P = g.P;
  a.KC = p.KC; a.Npad = p.Npad; a.nkg = p.nkg; a.G = p.G;
  a.L = p.L; a.nseg = p.nseg; a.nitems = p.nitems;
  a.pitch = p.pitch; a.rs_rows = p.rs_rows; a.rs_floats = p.rs_floats; a.stage_bytes = p.stage_bytes;
  a.dbg = 0;
  a.cpt = kWgMaxCpt;
  a.tdbg = nullptr;
  switch (p.Npad / 4) {
    case 4: return run_wgrad_tc<4>(tm, a, p.grid, p.smem, st);
    case 8: return run_wgrad_tc<8>(tm, a, p.grid, p.smem, st);
    case 12: return run_wgrad_tc<12>(tm, a, p.grid, p.smem, st);
    case 16: return run_wgrad_tc<16>(tm, a, p.grid, p.smem, st);
    case 20: return run_wgrad_tc<20>(tm, a, p.grid, p.smem, st);
    case 24: return run_wgrad_tc<24>(tm, a, p.grid, p.smem, st);
    case 28: return run_wgrad_tc<28>(tm, a, p.grid, p.smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace csc

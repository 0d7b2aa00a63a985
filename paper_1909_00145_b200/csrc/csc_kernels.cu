// csc_kernels.cu -- sm_100a kernels of the stochastic spatial-domain CSC hot path.
//
// Method: arxiv 1909.00145, PAPER.md (citations P:n = line n).  Readings
// R1..R9 / #1..#17: DESIGN.md §3.  Layouts: include/csc.h.
//
//   conv_fwd_kernel      r = sum_k d_k * z_k - x  (also Zg with g for d)
//   wgrad_kernel         g = Z^T r                 (gradient of the Eq.5 fit term)
//   code_step_kernel     masked prox-gradient step on the codes (Eq.2-4)
//   mask_*_kernel        Bernoulli(p) mask from counter-based Philox4x32-10 (Eq.2, R4/R5)
//   lipschitz_*_kernel   L_D on the 64x64 DFT grid (R8)
//   filter_*_kernel      exact line search + unit-ball projection (R6-R8)
//
// Everything is FP32 state with FP64 cross-thread/cross-block sums in a fixed
// order (deterministic run to run).  This file shares no code with oracle/.
#include "csc_internal.cuh"
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include <cstdint>
#include <cuda_runtime.h>

namespace csc {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void cp_async_f32(float* smem_dst, const float* gmem_src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int bytes = valid ? 4 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem_src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree, then warp partials in order).
// Result valid in thread 0.  Requires blockDim.x % 32 == 0, <= 1024.
__device__ double block_sum_d(double v) {
  __shared__ double red[32];
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) t += red[i];
  }
  return t;
}

__device__ double block_max_d(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; ++i) t = fmax(t, red[i]);
  }
  return t;
}

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32->64 multiplies
// with the Weyl key schedule.  Independent of oracle/ (pinned against it and,
// through it, against curand).
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
constexpr uint32_t kMaskTag = 0x4353434Du;  // 4th counter word, "CSCM" (#13)

__device__ __forceinline__ uint4 mask_block(uint64_t seed, uint32_t iter, uint64_t q) {
  return philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), iter, kMaskTag),
                       make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
}
__device__ __forceinline__ uint32_t pick(const uint4& w, int i) {
  return i == 0 ? w.x : (i == 1 ? w.y : (i == 2 ? w.z : w.w));
}
// Block-structured masks (E5): one draw per aligned block b = l >> 3 of 8 coordinates,
// word b & 3 of Philox(ctr = {q lo, q hi, t, kSectorTag}, q = b >> 2).  r[j] = draw of l0 + j.
constexpr uint32_t kSectorTag = 0x43534253u;  // "CSBS"
__device__ __forceinline__ uint4 sector_block(uint64_t seed, uint32_t iter, uint64_t q) {
  return philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), iter, kSectorTag),
                       make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
}
__device__ __forceinline__ void mask_rnd4(int mode, uint64_t seed, uint32_t iter, uint64_t l0, uint32_t r[4]) {
  if (mode == 1) {
    const uint64_t qa = (l0 >> 3) >> 2, qb = ((l0 + 3) >> 3) >> 2;
    const uint4 wa = sector_block(seed, iter, qa);
    const uint4 wb = qb != qa ? sector_block(seed, iter, qb) : wa;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t b = (l0 + j) >> 3;
      r[j] = pick((b >> 2) == qa ? wa : wb, static_cast<int>(b & 3));
    }
  } else {
    const uint64_t qa = l0 >> 2;
    const uint4 wa = mask_block(seed, iter, qa);
    const uint4 wb = (l0 & 3) != 0 ? mask_block(seed, iter, qa + 1) : wa;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t l = l0 + j;
      r[j] = pick((l >> 2) == qa ? wa : wb, static_cast<int>(l & 3));
    }
  }
}

// Canonical layout: one 32-bit word per thread, bit l = (k*Hc+u)*Wc+v.
__global__ void mask_bits_kernel(uint64_t total, uint64_t seed, uint32_t iter, uint64_t thr, int mode,
                                 uint32_t* __restrict__ bits) {
  const uint64_t wi = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nwords = (total + 31) / 32;
  if (wi >= nwords) return;
  uint32_t word = 0;
#pragma unroll 1
  for (int qq = 0; qq < 8; ++qq) {
    const uint64_t q = wi * 8 + qq;
    if (q * 4 >= total) break;
    uint32_t v[4];
    mask_rnd4(mode, seed, iter, q * 4, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t l = q * 4 + j;
      if (l < total && static_cast<uint64_t>(v[j]) < thr) word |= 1u << (qq * 4 + j);
    }
  }
  bits[wi] = word;
}

// Column-word layout for the code step: thread per (k, ub, quad of 4 columns);
// colw[(k*NB+ub)*Wc+v] bit r = mask(k, 32*ub+r, v).  Rows >= Hc are 0.
__global__ void mask_colwords_kernel(Geom g, int NB, uint64_t seed, uint32_t iter, const uint32_t* iter_off,
                                     uint64_t thr, int mode, uint32_t* __restrict__ colw) {
  if (iter_off != nullptr) iter += *iter_off;  // device-side step counter (CUDA-graph replays)
  const int nq = (g.Wc + 3) / 4;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(g.K) * NB * nq;
  if (tid >= total) return;
  const int vq = static_cast<int>(tid % nq);
  const int64_t kb = tid / nq;
  const int ub = static_cast<int>(kb % NB);
  const int k = static_cast<int>(kb / NB);
  const int v0 = vq * 4;
  uint32_t out[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
  for (int r = 0; r < 32; ++r) {
    const int u = ub * 32 + r;
    if (u >= g.Hc) break;
    const uint64_t l0 = (static_cast<uint64_t>(k) * g.Hc + u) * g.Wc + v0;
    uint32_t w4[4];
    mask_rnd4(mode, seed, iter, l0, w4);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (v0 + c >= g.Wc) break;
      if (static_cast<uint64_t>(w4[c]) < thr) out[c] |= 1u << r;
    }
  }
  uint32_t* dst = colw + (static_cast<int64_t>(k) * NB + ub) * g.Wc + v0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (v0 + c < g.Wc) dst[c] = out[c];
}

// ------------------------------------------------------------------ conv fwd
// y[n,i,j] = sum_{k in split} sum_{a,b} f[k,a,b] z[n,k,i+P-a,j+P-b]
// Tile 64x64 outputs, 128 threads, each thread a 4x8 register block.  The z
// halo tile (64+P)^2 and the filter are double-buffered in shared memory with
// cp.async; the filter tap row a for (z row rho, output row r_) is a = r_+P-rho.
template <int S>
struct ConvTile {
  static constexpr int P = S - 1;
  static constexpr int ZH = kConvTH + P;
  static constexpr int ZW = kConvTW + P;
  static constexpr int ZP = ((ZW + 3) / 4) * 4;
  static constexpr int FP = ((S + 3) / 4) * 4;
  static constexpr int ZR = ((kConvC + P + 3) / 4) * 4;
  static constexpr int ZTILE = ZH * ZP;
  static constexpr int FTILE = S * FP;
  static constexpr int SMEM_FLOATS = 2 * (ZTILE + FTILE);
};

template <int S>
__device__ __forceinline__ void conv_load_stage(float* zs, float* fs, const float* __restrict__ zk,
                                                const float* __restrict__ fk, const Geom& g, int i0, int j0) {
  using T = ConvTile<S>;
  for (int e = threadIdx.x; e < T::ZH * T::ZW; e += kConvThreads) {
    const int rr = e / T::ZW, cc = e - rr * T::ZW;
    const int u = i0 + rr, v = j0 + cc;
    const bool ok = (u < g.Hc) && (v < g.Wc);
    cp_async_f32(zs + rr * T::ZP + cc, ok ? zk + static_cast<int64_t>(u) * g.Wc + v : zk, ok);
  }
  for (int e = threadIdx.x; e < S * S; e += kConvThreads) {
    const int a = e / S, b = e - a * S;
    cp_async_f32(fs + a * T::FP + b, fk + e, true);
  }
}

template <int S>
__global__ void __launch_bounds__(kConvThreads, 4)
conv_fwd_kernel(const float* __restrict__ z, const float* __restrict__ filt, const float* __restrict__ x,
                float* __restrict__ out, int mode, int ksplit, Geom g, int tilesX,
                double* __restrict__ sq_part, double* __restrict__ l1_part) {
  using T = ConvTile<S>;
  constexpr int P = T::P;
  constexpr int R = kConvR, C = kConvC;
  extern __shared__ __align__(16) float smem[];
  float* zbuf[2] = {smem, smem + T::ZTILE};
  float* fbuf[2] = {smem + 2 * T::ZTILE, smem + 2 * T::ZTILE + T::FTILE};

  const int tile = blockIdx.x;
  const int n = blockIdx.y;
  const int ks = blockIdx.z;
  const int i0 = (tile / tilesX) * kConvTH;
  const int j0 = (tile % tilesX) * kConvTW;
  const int k0 = static_cast<int>((static_cast<int64_t>(ks) * g.K) / ksplit);
  const int k1 = static_cast<int>((static_cast<int64_t>(ks + 1) * g.K) / ksplit);
  const int tx = threadIdx.x % kConvTX, ty = threadIdx.x / kConvTX;
  const int64_t zimg = static_cast<int64_t>(n) * g.K * g.Hc * g.Wc;
  const int64_t kstride = static_cast<int64_t>(g.Hc) * g.Wc;

  // owned code positions for the L1 norm (each code counted once over all tiles)
  const int u_end = (i0 + kConvTH >= g.H) ? g.Hc : i0 + kConvTH;
  const int v_end = (j0 + kConvTW >= g.W) ? g.Wc : j0 + kConvTW;
  double l1 = 0.0;

  float acc[R][C];
#pragma unroll
  for (int r_ = 0; r_ < R; ++r_)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r_][c] = 0.f;

  if (k0 < k1) {
    conv_load_stage<S>(zbuf[0], fbuf[0], z + zimg + k0 * kstride, filt + static_cast<int64_t>(k0) * S * S, g, i0, j0);
    cp_async_commit();
  }
  for (int k = k0; k < k1; ++k) {
    const int buf = (k - k0) & 1;
    if (k + 1 < k1) {
      conv_load_stage<S>(zbuf[buf ^ 1], fbuf[buf ^ 1], z + zimg + (k + 1) * kstride,
                         filt + static_cast<int64_t>(k + 1) * S * S, g, i0, j0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* zs = zbuf[buf];
    const float* fs = fbuf[buf];
    if (l1_part != nullptr) {
      float s1 = 0.f;
      for (int e = threadIdx.x; e < T::ZH * T::ZW; e += kConvThreads) {
        const int rr = e / T::ZW, cc = e - rr * T::ZW;
        const int u = i0 + rr, v = j0 + cc;
        if (u < u_end && v < v_end) s1 += fabsf(zs[rr * T::ZP + cc]);
      }
      l1 += static_cast<double>(s1);
    }
    const float* zt = zs + (ty * R) * T::ZP + tx * C;
#pragma unroll 1
    for (int rho = 0; rho < R + P; ++rho) {
      float zr[T::ZR];
#pragma unroll
      for (int q = 0; q < T::ZR / 4; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(zt + rho * T::ZP + 4 * q);
        zr[4 * q + 0] = v4.x; zr[4 * q + 1] = v4.y; zr[4 * q + 2] = v4.z; zr[4 * q + 3] = v4.w;
      }
#pragma unroll
      for (int r_ = 0; r_ < R; ++r_) {
        const int a = r_ + P - rho;
        if (a >= 0 && a <= P) {
          float fr[T::FP];
#pragma unroll
          for (int q = 0; q < T::FP / 4; ++q) {
            const float4 v4 = *reinterpret_cast<const float4*>(fs + a * T::FP + 4 * q);
            fr[4 * q + 0] = v4.x; fr[4 * q + 1] = v4.y; fr[4 * q + 2] = v4.z; fr[4 * q + 3] = v4.w;
          }
#pragma unroll
          for (int b = 0; b < S; ++b)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r_][c] = fmaf(fr[b], zr[c + P - b], acc[r_][c]);
        }
      }
    }
    __syncthreads();
  }

  const int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  double sq = 0.0;
  const int64_t img = static_cast<int64_t>(n) * g.H * g.W;
  if (ksplit == 1) {
#pragma unroll
    for (int r_ = 0; r_ < R; ++r_) {
      const int i = i0 + ty * R + r_;
      if (i >= g.H) continue;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int j = j0 + tx * C + c;
        if (j >= g.W) continue;
        const int64_t idx = img + static_cast<int64_t>(i) * g.W + j;
        float v = acc[r_][c];
        if (mode == kConvResidual) {
          if (x != nullptr) v = v - x[idx];
          out[idx] = v;
        }
        sq += static_cast<double>(v) * static_cast<double>(v);
      }
    }
    const double t = block_sum_d(sq);
    if (threadIdx.x == 0 && sq_part != nullptr) sq_part[bid] = t;
  } else {
    float* dst = out + static_cast<int64_t>(ks) * g.N * g.H * g.W + img;
#pragma unroll
    for (int r_ = 0; r_ < R; ++r_) {
      const int i = i0 + ty * R + r_;
      if (i >= g.H) continue;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int j = j0 + tx * C + c;
        if (j < g.W) dst[static_cast<int64_t>(i) * g.W + j] = acc[r_][c];
      }
    }
  }
  if (l1_part != nullptr) {
    const double t = block_sum_d(l1);
    if (threadIdx.x == 0) l1_part[bid] = t;
  }
}

__global__ void conv_finalize_kernel(const float* __restrict__ part, int ksplit, int64_t npix,
                                     const float* __restrict__ x, float* __restrict__ r, int mode,
                                     double* __restrict__ sq_part) {
  double sq = 0.0;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < npix;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v = 0.f;
    for (int ks = 0; ks < ksplit; ++ks) v += part[ks * npix + idx];
    if (mode == kConvResidual) {
      if (x != nullptr) v = v - x[idx];
      r[idx] = v;
    }
    sq += static_cast<double>(v) * static_cast<double>(v);
  }
  const double t = block_sum_d(sq);
  if (threadIdx.x == 0) sq_part[blockIdx.x] = t;
}

__global__ void reduce_sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out,
                                  double scale) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  const double t = block_sum_d(s);
  if (threadIdx.x == 0) *out = t * scale;
}

// ------------------------------------------------------------------ wgrad
// g[k,a,b] = sum_n sum_ij r[n,i,j] z[n,k,i+P-a,j+P-b].  Grid (G, K): the CTA for
// (gi, k) loops over tiles t = gi, gi+G, ... of all images, accumulating the
// full s x s tap block per thread in registers; one fixed-order reduction at the end.
template <int S>
struct WgTile {
  static constexpr int P = S - 1;
  static constexpr int ZH = kWgTH + P;
  static constexpr int ZW = kWgTW + P;
  static constexpr int ZP = ((ZW + 3) / 4) * 4;
  static constexpr int RP = kWgTW;
  static constexpr int ZR = ((kWgC + P + 3) / 4) * 4;
  static constexpr int SMEM_FLOATS = ZH * ZP + kWgTH * RP;
};

template <int S>
__global__ void __launch_bounds__(kWgThreads, 2)
wgrad_kernel(const float* __restrict__ z, const float* __restrict__ r, Geom g, int tilesX, int tilesY,
             int G, double* __restrict__ gpart) {
  using T = WgTile<S>;
  constexpr int P = T::P;
  constexpr int C = kWgC, RB = kWgRB;
  extern __shared__ __align__(16) float smem[];
  float* zs = smem;
  float* rs = smem + T::ZH * T::ZP;
  const int gi = blockIdx.x, k = blockIdx.y;
  const int tx = threadIdx.x % kWgTX, ty = threadIdx.x / kWgTX;
  const int ntiles = g.N * tilesX * tilesY;

  float acc[S][S];
#pragma unroll
  for (int a = 0; a < S; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) acc[a][b] = 0.f;

  for (int t = gi; t < ntiles; t += G) {
    const int n = t / (tilesX * tilesY);
    const int tt = t - n * tilesX * tilesY;
    const int i0 = (tt / tilesX) * kWgTH, j0 = (tt % tilesX) * kWgTW;
    const float* zk = z + (static_cast<int64_t>(n) * g.K + k) * g.Hc * g.Wc;
    const float* rn = r + static_cast<int64_t>(n) * g.H * g.W;
    __syncthreads();
    for (int e = threadIdx.x; e < T::ZH * T::ZW; e += kWgThreads) {
      const int rr = e / T::ZW, cc = e - rr * T::ZW;
      const int u = i0 + rr, v = j0 + cc;
      const bool ok = (u < g.Hc) && (v < g.Wc);
      cp_async_f32(zs + rr * T::ZP + cc, ok ? zk + static_cast<int64_t>(u) * g.Wc + v : zk, ok);
    }
    for (int e = threadIdx.x; e < kWgTH * kWgTW; e += kWgThreads) {
      const int rr = e / kWgTW, cc = e - rr * kWgTW;
      const int i = i0 + rr, j = j0 + cc;
      const bool ok = (i < g.H) && (j < g.W);
      cp_async_f32(rs + rr * T::RP + cc, ok ? rn + static_cast<int64_t>(i) * g.W + j : rn, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll 1
    for (int rr = 0; rr < RB; ++rr) {
      const int il = ty * RB + rr;
      float rv[C];
#pragma unroll
      for (int q = 0; q < C / 4; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(rs + il * T::RP + tx * C + 4 * q);
        rv[4 * q + 0] = v4.x; rv[4 * q + 1] = v4.y; rv[4 * q + 2] = v4.z; rv[4 * q + 3] = v4.w;
      }
      const float* zrow0 = zs + (il + P) * T::ZP + tx * C;
#pragma unroll
      for (int a = 0; a < S; ++a) {
        float zr[T::ZR];
#pragma unroll
        for (int q = 0; q < T::ZR / 4; ++q) {
          const float4 v4 = *reinterpret_cast<const float4*>(zrow0 - a * T::ZP + 4 * q);
          zr[4 * q + 0] = v4.x; zr[4 * q + 1] = v4.y; zr[4 * q + 2] = v4.z; zr[4 * q + 3] = v4.w;
        }
#pragma unroll
        for (int b = 0; b < S; ++b)
#pragma unroll
          for (int c = 0; c < C; ++c) acc[a][b] = fmaf(rv[c], zr[c + P - b], acc[a][b]);
      }
    }
  }

  // fixed-order reduction of the per-thread tap blocks
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem);  // [warps][S*S]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int a = 0; a < S; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) {
      const double v = warp_sum_d(static_cast<double>(acc[a][b]));
      if (l == 0) red[w * S * S + a * S + b] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < S * S; e += kWgThreads) {
    double s = 0.0;
    for (int ww = 0; ww < kWgThreads / 32; ++ww) s += red[ww * S * S + e];
    gpart[(static_cast<int64_t>(gi) * g.K + k) * S * S + e] = s;
  }
}

// 32 elements x 8 partial slices per 256-thread block: slice y sums partials y, y+8, ... (4 loads in
// flight), then the 8 slice sums are added in slice order -- a fixed order, so the result is deterministic
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const double* __restrict__ gpart, int G, int nel,
                                                           double* __restrict__ gsum) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + tx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (e < nel) {
    int gi = ty;
    for (; gi + 24 < G; gi += 32) {
      s0 += __ldg(gpart + static_cast<int64_t>(gi) * nel + e);
      s1 += __ldg(gpart + static_cast<int64_t>(gi + 8) * nel + e);
      s2 += __ldg(gpart + static_cast<int64_t>(gi + 16) * nel + e);
      s3 += __ldg(gpart + static_cast<int64_t>(gi + 24) * nel + e);
    }
    for (; gi < G; gi += 8) s0 += __ldg(gpart + static_cast<int64_t>(gi) * nel + e);
  }
  red[ty][tx] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (ty == 0 && e < nel) {
    double s = red[0][tx];
#pragma unroll
    for (int y = 1; y < 8; ++y) s += red[y][tx];
    gsum[e] = s;
  }
}

// g32 = fp32(g) and <g, g>: one element per thread, block sums into scratch[blockIdx.x], and the last
// block adds the block sums in block order (deterministic) into *gg_out and clears the block counter
// (scratch[gridDim.x], zero at allocation)
__global__ void __launch_bounds__(256) grad_finish_kernel(const double* __restrict__ gsum, int nel,
                                                         float* __restrict__ g32, double* __restrict__ gg_out,
                                                         double* __restrict__ scratch) {
  __shared__ bool last;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (i < nel) {
    const double v = gsum[i];
    g32[i] = static_cast<float>(v);
    s = v * v;
  }
  const double t = block_sum_d(s);
  if (threadIdx.x == 0) {
    scratch[blockIdx.x] = t;
    __threadfence();
    auto* cnt = reinterpret_cast<unsigned long long*>(scratch + gridDim.x);
    last = atomicAdd(cnt, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double tot = 0.0;
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) tot += __ldcg(scratch + b);
    *gg_out = tot;
    *reinterpret_cast<unsigned long long*>(scratch + gridDim.x) = 0ull;
  }
}

// ------------------------------------------------------------------ code step
// CTA = (32-column strip, TH-row band, image n, k group); lane L owns column
// v0+L; the 4 warps take k = kb+w, kb+w+4, ...  Each lane walks the masked rows
// of its column (bits from the column-word mask) and, per masked code, does the
// s^2-tap correlation with the residual tile in shared memory (pitch 64 => the
// 32 lanes always hit 32 distinct banks), the step and the shrinkage.  Codes
// whose value does not change are not written back.
template <int S>
__global__ void __launch_bounds__(kCodeThreads, 3)
code_step_kernel(const float* __restrict__ r, const float* __restrict__ d, float* __restrict__ z,
                 const uint32_t* __restrict__ colw, int all_selected, const float* __restrict__ tau_dev,
                 int tau_stride, float lam, Geom g, int TH, int kgroups, int NB, uint32_t* __restrict__ zmax) {
  constexpr int P = S - 1;
  extern __shared__ __align__(16) float rs[];
  const int v0 = blockIdx.x * 32;
  const int u0 = blockIdx.y * TH;
  const int n = blockIdx.z / kgroups;
  const int kg = blockIdx.z - n * kgroups;
  const int kb = static_cast<int>((static_cast<int64_t>(kg) * g.K) / kgroups);
  const int ke = static_cast<int>((static_cast<int64_t>(kg + 1) * g.K) / kgroups);
  const float* rn = r + static_cast<int64_t>(n) * g.H * g.W;

  // residual tile: rows [u0-P, u0+TH), cols [v0-P, v0+32), zero outside the image
  const int tw = 32 + P;
  for (int e = threadIdx.x; e < (TH + P) * tw; e += kCodeThreads) {
    const int lr = e / tw, lc = e - lr * tw;
    const int i = u0 - P + lr, j = v0 - P + lc;
    float v = 0.f;
    if (i >= 0 && i < g.H && j >= 0 && j < g.W) v = rn[static_cast<int64_t>(i) * g.W + j];
    rs[lr * kCodePitch + lc] = v;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = v0 + lane;
  const bool col_ok = v < g.Wc;
  const int nblk = TH / 32;
  const int ub0 = u0 / 32;
  float wmax = 0.f;

  for (int k = kb + warp; k < ke; k += kCodeWarps) {
    const float tau = tau_dev[k * tau_stride];
    const float kappa = tau * lam;
    float dk[S * S];
#pragma unroll
    for (int i = 0; i < S * S; ++i) dk[i] = __ldg(d + static_cast<int64_t>(k) * S * S + i);
    uint32_t q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ub = ub0 + j;
      uint32_t wbits = 0u;
      if (j < nblk && ub < NB && col_ok) {
        if (all_selected) {
          const int rows = g.Hc - ub * 32;
          wbits = rows >= 32 ? kFull : ((1u << rows) - 1u);
        } else {
          wbits = __ldg(colw + (static_cast<int64_t>(k) * NB + ub) * g.Wc + v);
        }
      }
      q[j] = wbits;
    }
    float* zk = z + (static_cast<int64_t>(n) * g.K + k) * g.Hc * g.Wc;
    uint32_t bits = q[0];
    int blk = 0;
    while (true) {
      while (bits == 0u && blk < 3) {
        bits = q[1]; q[1] = q[2]; q[2] = q[3]; q[3] = 0u; ++blk;
      }
      const bool have = bits != 0u;
      if (!__any_sync(kFull, have)) break;
      if (have) {
        const int rbit = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int ul = blk * 32 + rbit;
        const int u = u0 + ul;
        const int64_t zi = static_cast<int64_t>(u) * g.Wc + v;
        const float zv = zk[zi];
        const float* rp = rs + ul * kCodePitch + lane;
        float c = 0.f;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int b = 0; b < S; ++b) c = fmaf(dk[a * S + b], rp[a * kCodePitch + b], c);
        const float w = fmaf(-tau, c, zv);
        const float nz = (w > kappa) ? (w - kappa) : ((w < -kappa) ? (w + kappa) : 0.f);
        if (nz != zv) {
          zk[zi] = nz;
          wmax = fmaxf(wmax, fabsf(nz));
        }
      }
    }
  }
  uint32_t wb = __float_as_uint(wmax);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wb = max(wb, __shfl_xor_sync(kFull, wb, o));
  if (lane == 0 && zmax != nullptr && wb != 0u) atomicMax(zmax, wb);
}

// ------------------------------------------------------------------ Lipschitz
// part[kc][m1*64+m2] = sum_{k in chunk kc} |d^_k(m1, m2)|^2, d^_k(m1,m2) = sum_{a,b} d[k,a,b] w^(a m1 + b m2),
// w = e^{-2 pi i/64}, evaluated separably: R[k][a][m2] = sum_b d[k,a,b] w^(b m2) (shared memory), then
// d^_k(m1,m2) = sum_a R[k][a][m2] w^(a m1).  Block = kLipKChunk filters, thread = 16 grid points.
constexpr int kLipG = 64;
constexpr int kLipKChunk = 2;
constexpr int kLipThreads = 256;
__global__ void __launch_bounds__(kLipThreads) lipschitz_partial_kernel(const float* __restrict__ d, Geom g,
                                                                      double* __restrict__ part) {
  __shared__ double twc[kLipG], tws[kLipG];
  __shared__ double rre[kLipKChunk][11][kLipG], rim[kLipKChunk][11][kLipG];
  const int kc = blockIdx.x;
  const int S = g.S;
  const int k0 = kc * kLipKChunk, k1 = min(g.K, k0 + kLipKChunk);
  if (threadIdx.x < kLipG) {
    double sv, cv;
    sincospi(-2.0 * static_cast<double>(threadIdx.x) / kLipG, &sv, &cv);
    twc[threadIdx.x] = cv;
    tws[threadIdx.x] = sv;
  }
  __syncthreads();
  // row transforms
  for (int e = threadIdx.x; e < (k1 - k0) * S * kLipG; e += kLipThreads) {
    const int m2 = e % kLipG;
    const int r = e / kLipG;
    const int a = r % S, kk = r / S;
    const float* da = d + (static_cast<int64_t>(k0 + kk) * S + a) * S;
    double re = 0.0, im = 0.0;
    for (int b = 0; b < S; ++b) {
      const double dv = static_cast<double>(__ldg(da + b));
      const int idx = (b * m2) & (kLipG - 1);
      re += dv * twc[idx];
      im += dv * tws[idx];
    }
    rre[kk][a][m2] = re;
    rim[kk][a][m2] = im;
  }
  __syncthreads();
  // grid.y splits the 64x64 grid points so that K/2 filter chunks still fill the GPU
  const int npt = kLipG * kLipG / gridDim.y;
  for (int pt = blockIdx.y * npt + threadIdx.x; pt < (blockIdx.y + 1) * npt; pt += kLipThreads) {
    const int m1 = pt / kLipG, m2 = pt % kLipG;
    double tot = 0.0;
    for (int kk = 0; kk < k1 - k0; ++kk) {
      double re = 0.0, im = 0.0;
      for (int a = 0; a < S; ++a) {
        const int ia = (a * m1) & (kLipG - 1);
        const double c = twc[ia], sn = tws[ia];
        const double ra = rre[kk][a][m2], ib = rim[kk][a][m2];
        re += ra * c - ib * sn;
        im += ra * sn + ib * c;
      }
      tot += re * re + im * im;
    }
    part[static_cast<int64_t>(kc) * kLipG * kLipG + pt] = tot;
  }
}

// One kernel for the sum over filter chunks and the max: block = 64 grid points x 4 chunk ranges of the
// filter-chunk partials (each summed in order, then the 4 in order: a fixed order), the block max into
// a 64-bit atomic max (non-negative doubles order as their bits), the last block writes L and 1/L and
// clears the max and the block counter for the next launch (state[0] = max bits, state[1] = count).
__global__ void __launch_bounds__(256) lipschitz_final2_kernel(const double* __restrict__ part, int nkc,
                                                              unsigned long long* __restrict__ state,
                                                              double* __restrict__ lhat, float* __restrict__ tau_out) {
  __shared__ double ps[4][64];
  __shared__ bool last;
  const int pl = threadIdx.x & 63, ch = threadIdx.x >> 6;
  const int pt = blockIdx.x * 64 + pl;
  const int per = (nkc + 3) / 4;
  const int c0 = ch * per, c1 = min(nkc, c0 + per);
  double s = 0.0;
#pragma unroll 8
  for (int kc = c0; kc < c1; ++kc) s += __ldg(part + static_cast<int64_t>(kc) * kLipG * kLipG + pt);
  ps[ch][pl] = s;
  __syncthreads();
  double m = 0.0;
  if (threadIdx.x < 64) {
    m = ((ps[0][pl] + ps[1][pl]) + ps[2][pl]) + ps[3][pl];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if (threadIdx.x == 0) ps[0][0] = m;
  __syncthreads();
  if (threadIdx.x == 32) ps[0][0] = fmax(ps[0][0], m);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(state, static_cast<unsigned long long>(__double_as_longlong(ps[0][0])));
    __threadfence();
    last = atomicAdd(state + 1, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const double L = __longlong_as_double(static_cast<long long>(atomicAdd(state, 0ull)));
    *lhat = L;
    if (tau_out != nullptr) *tau_out = L > 0.0 ? static_cast<float>(1.0 / L) : 0.f;
    state[0] = 0ull;
    state[1] = 0ull;
  }
}


// ------------------------------------------------------------------ filter update
__global__ void filter_tau_kernel(const double* __restrict__ gg, const double* __restrict__ zg2, float step,
                                  float* __restrict__ tau_d) {
  if (step > 0.f) {
    *tau_d = step;
  } else {
    const double den = *zg2;
    *tau_d = den > 0.0 ? static_cast<float>(*gg / den) : 0.f;
  }
}

__global__ void filter_update_kernel(float* __restrict__ d, const double* __restrict__ gsum,
                                     const float* __restrict__ tau_d, int M) {
  const int k = blockIdx.x;
  const double tau = static_cast<double>(*tau_d);
  double e_loc[8];
  double s2 = 0.0;
  int cnt = 0;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const double e = static_cast<double>(d[static_cast<int64_t>(k) * M + i]) - tau * gsum[static_cast<int64_t>(k) * M + i];
    e_loc[cnt++] = e;
    s2 += e * e;
  }
  __shared__ double scale_sh;
  const double t = block_sum_d(s2);
  if (threadIdx.x == 0) scale_sh = fmax(1.0, sqrt(t));
  __syncthreads();
  const double scale = scale_sh;
  cnt = 0;
  for (int i = threadIdx.x; i < M; i += blockDim.x) d[static_cast<int64_t>(k) * M + i] = static_cast<float>(e_loc[cnt++] / scale);
}

__global__ void neg_copy_kernel(const float* __restrict__ x, float* __restrict__ r, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    r[i] = -x[i];
}

template <template <int> class F, typename... Args>
cudaError_t dispatch_s(int s, Args&&... args) {
  switch (s) {
    case 1: return F<1>::run(args...);
    case 3: return F<3>::run(args...);
    case 5: return F<5>::run(args...);
    case 7: return F<7>::run(args...);
    case 9: return F<9>::run(args...);
    case 11: return F<11>::run(args...);
    default: return cudaErrorInvalidValue;
  }
}

template <int S>
struct ConvRun {
  static cudaError_t run(const Geom& g, const float* z, const float* filt, const float* x, float* out, int ksplit,
                         int mode, double* sq_part, double* l1_part, cudaStream_t st) {
    using T = ConvTile<S>;
    const int tilesX = ceil_div(g.W, kConvTW), tilesY = ceil_div(g.H, kConvTH);
    const size_t smem = sizeof(float) * T::SMEM_FLOATS;
    cudaError_t ea = set_smem_attr_once(reinterpret_cast<const void*>(&conv_fwd_kernel<S>), static_cast<int>(smem));
    if (ea != cudaSuccess) return ea;
    dim3 grid(tilesX * tilesY, g.N, ksplit);
    conv_fwd_kernel<S><<<grid, kConvThreads, smem, st>>>(z, filt, x, out, mode, ksplit, g, tilesX, sq_part, l1_part);
    return cudaGetLastError();
  }
};

template <int S>
struct WgRun {
  static cudaError_t run(const Geom& g, const float* z, const float* r, int G, double* gpart, cudaStream_t st) {
    using T = WgTile<S>;
    const int tilesX = ceil_div(g.W, kWgTW), tilesY = ceil_div(g.H, kWgTH);
    size_t smem = sizeof(float) * T::SMEM_FLOATS;
    const size_t red = sizeof(double) * (kWgThreads / 32) * S * S;
    if (red > smem) smem = red;
    cudaError_t ea = set_smem_attr_once(reinterpret_cast<const void*>(&wgrad_kernel<S>), static_cast<int>(smem));
    if (ea != cudaSuccess) return ea;
    dim3 grid(G, g.K);
    wgrad_kernel<S><<<grid, kWgThreads, smem, st>>>(z, r, g, tilesX, tilesY, G, gpart);
    return cudaGetLastError();
  }
};

inline int code_tile_rows(int Hc) {
  // rows per band: a multiple of 32 (column words are 32-row aligned), <= 128,
  // chosen to minimise padding rows.
  int best = 32, best_waste = 1 << 30;
  for (int th = 32; th <= 128; th += 32) {
    const int waste = ceil_div(Hc, th) * th - Hc;
    if (waste < best_waste || (waste == best_waste && th > best)) {
      best = th;
      best_waste = waste;
    }
  }
  return best;
}

template <int S>
struct CodeRun {
  static cudaError_t run(const Geom& g, const float* r, const float* d, float* z, const uint32_t* colw,
                         int all_selected, const float* tau_dev, int tau_stride, float lam, uint32_t* zmax,
                         cudaStream_t st) {
    const int TH = code_tile_rows(g.Hc);
    const int strips = ceil_div(g.Wc, 32), bands = ceil_div(g.Hc, TH);
    const int base = strips * bands * g.N;
    int kgroups = ceil_div(148 * 6, base > 0 ? base : 1);
    const int kmax = ceil_div(g.K, kCodeWarps);
    if (kgroups > kmax) kgroups = kmax;
    if (kgroups < 1) kgroups = 1;
    const size_t smem = sizeof(float) * (TH + S - 1) * kCodePitch;
    cudaError_t ea = set_smem_attr_once(reinterpret_cast<const void*>(&code_step_kernel<S>), 96 * 1024);
    if (ea != cudaSuccess) return ea;
    const int NB = ceil_div(g.Hc, 32);
    dim3 grid(strips, bands, g.N * kgroups);
    code_step_kernel<S><<<grid, kCodeThreads, smem, st>>>(r, d, z, colw, all_selected, tau_dev, tau_stride, lam, g,
                                                          TH, kgroups, NB, zmax);
    return cudaGetLastError();
  }
};

}  // namespace

// ------------------------------------------------------------------ launchers
int conv_fwd_blocks(const Geom& g, int ksplit) {
  return ceil_div(g.W, kConvTW) * ceil_div(g.H, kConvTH) * g.N * ksplit;
}

cudaError_t launch_conv_fwd(const Geom& g, const float* z, const float* filt, const float* x, float* r,
                            float* part, int ksplit, int mode, double* sq_part, double* l1_part,
                            cudaStream_t st, int* nblocks_out) {
  if (nblocks_out) *nblocks_out = conv_fwd_blocks(g, ksplit);
  float* out = ksplit == 1 ? r : part;
  return dispatch_s<ConvRun>(g.S, g, z, filt, x, out, ksplit, mode, sq_part, l1_part, st);
}

cudaError_t launch_conv_finalize(const Geom& g, const float* part, int ksplit, const float* x, float* r, int mode,
                                 double* sq_part, cudaStream_t st) {
  const int64_t npix = static_cast<int64_t>(g.N) * g.H * g.W;
  conv_finalize_kernel<<<kFinalizeBlocks, 256, 0, st>>>(part, ksplit, npix, x, r, mode, sq_part);
  return cudaGetLastError();
}

cudaError_t launch_reduce_sum(const double* part, int n, double* out, double scale, cudaStream_t st) {
  reduce_sum_kernel<<<1, kReduceThreads, 0, st>>>(part, n, out, scale);
  return cudaGetLastError();
}

cudaError_t launch_wgrad(const Geom& g, const float* z, const float* r, int G, double* gpart, cudaStream_t st) {
  return dispatch_s<WgRun>(g.S, g, z, r, G, gpart, st);
}

cudaError_t launch_wgrad_reduce(const Geom& g, const double* gpart, int G, double* gsum, cudaStream_t st) {
  const int nel = g.K * g.S * g.S;
  wgrad_reduce_kernel<<<ceil_div(nel, 32), 256, 0, st>>>(gpart, G, nel, gsum);
  return cudaGetLastError();
}

cudaError_t launch_grad_finish(const Geom& g, const double* gsum, float* g32, double* gg_out, double* scratch,
                               cudaStream_t st) {
  const int nel = g.K * g.S * g.S;
  grad_finish_kernel<<<ceil_div(nel, 256), 256, 0, st>>>(gsum, nel, g32, gg_out, scratch);
  return cudaGetLastError();
}

cudaError_t launch_mask_colwords(const Geom& g, uint64_t seed, uint32_t iter, uint64_t thr, uint32_t* colw,
                                 cudaStream_t st, int mode, const uint32_t* iter_off) {
  const int NB = ceil_div(g.Hc, 32);
  const int64_t total = static_cast<int64_t>(g.K) * NB * ceil_div(g.Wc, 4);
  mask_colwords_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(g, NB, seed, iter, iter_off, thr,
                                                                                    mode, colw);
  return cudaGetLastError();
}

cudaError_t launch_mask_bits(const Geom& g, uint64_t seed, uint32_t iter, uint64_t thr, uint32_t* bits,
                             cudaStream_t st, int mode) {
  const uint64_t total = static_cast<uint64_t>(g.K) * g.Hc * g.Wc;
  const uint64_t nwords = (total + 31) / 32;
  mask_bits_kernel<<<static_cast<unsigned>((nwords + 255) / 256), 256, 0, st>>>(total, seed, iter, thr, mode, bits);
  return cudaGetLastError();
}

cudaError_t launch_code_step(const Geom& g, const float* r, const float* d, float* z, const uint32_t* colw,
                             int all_selected, const float* tau_dev, float lam, uint32_t* zmax, cudaStream_t st,
                             int tau_stride) {
  return dispatch_s<CodeRun>(g.S, g, r, d, z, colw, all_selected, tau_dev, tau_stride, lam, zmax, st);
}

// ESO step rule (E1): tau_k = fp32(1 / (p L + (1-p) ||d_k||^2)), ||d_k||^2 summed in fp64
// over (a, b) in order; one thread per filter
__global__ void eso_tau_kernel(const float* __restrict__ d, int K, int S2, double p, const double* __restrict__ lhat,
                               float* __restrict__ tauk) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double dk2 = 0.0;
  for (int i = 0; i < S2; ++i) {
    const double v = static_cast<double>(d[static_cast<int64_t>(k) * S2 + i]);
    dk2 += v * v;
  }
  tauk[k] = static_cast<float>(1.0 / (p * *lhat + (1.0 - p) * dk2));
}

cudaError_t launch_eso_tau(const Geom& g, const float* d, double p, const double* lhat, float* tauk, cudaStream_t st) {
  eso_tau_kernel<<<ceil_div(g.K, 128), 128, 0, st>>>(d, g.K, g.S * g.S, p, lhat, tauk);
  return cudaGetLastError();
}

cudaError_t launch_lipschitz(const Geom& g, const float* d, double* part, double* lhat, float* tau_out,
                             cudaStream_t st) {
  const int nkc = ceil_div(g.K, kLipKChunk);
  lipschitz_partial_kernel<<<dim3(nkc, 4), kLipThreads, 0, st>>>(d, g, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // lip_part has 64 doubles of room past the partials (see csc_init): the final kernel's max / counter
  // state, zero at allocation and cleared by each launch's last block
  auto* state = reinterpret_cast<unsigned long long*>(part + static_cast<int64_t>(nkc) * kLipG * kLipG);
  lipschitz_final2_kernel<<<kLipG * kLipG / 64, 256, 0, st>>>(part, nkc, state, lhat, tau_out);
  return cudaGetLastError();
}

cudaError_t launch_filter_tau(const double* gg, const double* zg2, float step, float* tau_d, cudaStream_t st) {
  filter_tau_kernel<<<1, 1, 0, st>>>(gg, zg2, step, tau_d);
  return cudaGetLastError();
}

cudaError_t launch_filter_update(const Geom& g, float* d, const double* gsum, const float* tau_d, cudaStream_t st) {
  const int M = g.S * g.S;  // <= 121 <= 128 threads * 8 slots
  filter_update_kernel<<<g.K, 128, 0, st>>>(d, gsum, tau_d, M);
  return cudaGetLastError();
}

// r += sign * x (the residual moved to new images without a dense pass, csc_iterate)
__global__ void axpy_sign_kernel(const float* __restrict__ x, float* __restrict__ r, int64_t n, float sign) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    r[i] = fmaf(sign, x[i], r[i]);
}

// number of nonzero entries (csc_count_nonzero; the trace's nnz column): per-warp ballot counts, one
// 64-bit atomic per block
__global__ void __launch_bounds__(256) count_nonzero_kernel(const float* __restrict__ v, int64_t n,
                                                            unsigned long long* __restrict__ out) {
  __shared__ unsigned int wsum[8];
  unsigned int c = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += v[i] != 0.f ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < 8; ++w) t += wsum[w];
    atomicAdd(out, t);
  }
}

cudaError_t launch_count_nonzero(const float* v, int64_t n, uint64_t* out, cudaStream_t st) {
  count_nonzero_kernel<<<kFinalizeBlocks * 4, 256, 0, st>>>(v, n, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

// new images from a staging buffer with the residual moved along (csc_iterate_staged): r += x_old - x_new,
// x <- x_new in one pass (float4 when every pointer is 16-B aligned and n % 4 == 0)
__global__ void stage_swap_kernel(const float* __restrict__ xn, float* __restrict__ x, float* __restrict__ r,
                                  int64_t n, int shift, int vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vec) {
    const float4* xn4 = reinterpret_cast<const float4*>(xn);
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* r4 = reinterpret_cast<float4*>(r);
    for (int64_t i = t0; i < n / 4; i += stride) {
      const float4 a = xn4[i];
      if (shift) {
        const float4 o = x4[i];
        float4 rv = r4[i];
        rv.x = (rv.x + o.x) - a.x; rv.y = (rv.y + o.y) - a.y; rv.z = (rv.z + o.z) - a.z; rv.w = (rv.w + o.w) - a.w;
        r4[i] = rv;
      }
      x4[i] = a;
    }
    return;
  }
  for (int64_t i = t0; i < n; i += stride) {
    const float a = xn[i];
    if (shift) r[i] = (r[i] + x[i]) - a;
    x[i] = a;
  }
}

cudaError_t launch_stage_swap(const float* xn, float* x, float* r, int64_t n, bool shift, cudaStream_t st) {
  const int vec = ((reinterpret_cast<uintptr_t>(xn) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r)) & 15u) == 0 &&
                          n % 4 == 0
                      ? 1
                      : 0;
  stage_swap_kernel<<<kFinalizeBlocks, 256, 0, st>>>(xn, x, r, n, shift ? 1 : 0, vec);
  return cudaGetLastError();
}

cudaError_t launch_resid_shift(const float* x, float* r, int64_t n, float sign, cudaStream_t st) {
  axpy_sign_kernel<<<kFinalizeBlocks, 256, 0, st>>>(x, r, n, sign);
  return cudaGetLastError();
}

cudaError_t launch_neg_copy(const float* x, float* r, int64_t n, cudaStream_t st) {
  neg_copy_kernel<<<kFinalizeBlocks, 256, 0, st>>>(x, r, n);
  return cudaGetLastError();
}

}  // namespace csc

// ---------------------------------------------------------------- TMA maps and launch attributes
namespace csc {
namespace {
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_t encode_tiled() {
  static std::once_flag once;
  static PFN_encodeTiled_t fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}
std::mutex g_attr_mu;
}  // namespace

bool tmap_available() { return encode_tiled() != nullptr; }

cudaError_t tmap_2d(TmapCache& c, CUtensorMapDataType dt, const void* ptr, uint64_t d0, uint64_t d1, uint64_t stride1,
                    uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw, CUtensorMapL2promotion promo) {
  const uint64_t key[4] = {d0, d1, stride1,
                           (static_cast<uint64_t>(b0) << 32) | (static_cast<uint64_t>(b1) << 8) |
                               (static_cast<uint64_t>(sw) << 4) | static_cast<uint64_t>(dt)};
  if (c.valid && c.ptr == ptr && std::memcmp(c.key, key, sizeof(key)) == 0) return cudaSuccess;
  PFN_encodeTiled_t enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {stride1};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t estr[2] = {1u, 1u};
  CUresult cr = enc(&c.map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    c.valid = false;
    return cudaErrorInvalidValue;
  }
  c.ptr = ptr;
  std::memcpy(c.key, key, sizeof(key));
  c.valid = true;
  return cudaSuccess;
}

cudaError_t set_smem_attr_once(const void* func, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::vector<std::pair<const void*, int>> done;  // (function, device) pairs configured
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (const auto& d : done)
    if (d.first == func && d.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(func, dev);
  return e;
}

}  // namespace csc

// ---------------------------------------------------------------- device scalars
namespace csc {
namespace {
__global__ void set_f32_kernel(float* p, float v) { *p = v; }
__global__ void bcast_f32_kernel(float* dst, const float* src, int n) {
  const float v = *src;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = v;
}
}  // namespace
cudaError_t launch_set_f32(float* p, float v, cudaStream_t st) {
  set_f32_kernel<<<1, 1, 0, st>>>(p, v);
  return cudaGetLastError();
}
cudaError_t launch_bcast_f32(float* dst, const float* src, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  bcast_f32_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}
}  // namespace csc

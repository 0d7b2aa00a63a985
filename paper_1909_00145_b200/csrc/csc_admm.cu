// csc_admm.cu -- kernels of the ADMM masked-LASSO code solver (PAPER.md
// P:303-321 §3.2): the paper's own code update, as an alternative to the one-step prox-gradient
// code step of the hot path (reading R1).  The iteration itself is in csc_api.cu
// (csc_code_step_admm); DESIGN.md §9 has the readings A1-A7 and the cost model.
//
// Layout.  The mask M^t (Eq.2) is shared by all images (R3), so its selected positions are
// compacted ONCE into idx[0..mc) (ascending l = (k*Hc + u)*Wc + v) and every ADMM / CG vector is
// stored compact, [N][ms] fp32 (ms = mc rounded up to 4, pads held at 0): the vector work and its
// HBM traffic scale with p (the paper's 1/p reduction), not with the code volume.
// The operator A = D M^T runs as
//   expand (compact -> dense code buffer Zd, zeros off the mask, full coalesced lines) -> the
//   dense pass of the hot path,
// and A^T e as a gather over the s x s taps of each selected code (masked_dtr_kernel).
// CG scalars are per image, reduced in fp64 in a fixed order (deterministic), and stay on the
// device.
#include "csc_internal.cuh"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

namespace csc {
namespace {

constexpr unsigned kFullA = 0xffffffffu;
constexpr int kAT = 256;          // threads of the vector kernels
constexpr int kIdxWords = 1024;   // mask words per block of the index build

__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullA, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// sum of part[n][0..nb) in a fixed order (warp 0: lane-strided partial sums, then a fixed
// butterfly), broadcast to the block through smem
__device__ __forceinline__ double image_total(const double* __restrict__ part, int n, int nb, double* slot) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += part[static_cast<int64_t>(n) * nb + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullA, s, o);
    if (threadIdx.x == 0) *slot = s;
  }
  __syncthreads();
  return *slot;
}

// max over the block of mx (every thread calls it), then one global atomicMax per block: per-warp
// atomics on a single address serialise at L2 (~20k of them in a full expansion)
__device__ __forceinline__ void block_atomic_max(uint32_t mx, uint32_t* bound) {
  __shared__ uint32_t red;
  if (threadIdx.x == 0) red = 0u;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFullA, mx, o));
  if ((threadIdx.x & 31) == 0 && mx != 0u) atomicMax(&red, mx);
  __syncthreads();
  if (threadIdx.x == 0 && bound != nullptr && red != 0u) atomicMax(bound, red);
}

// ---- index build: idx[m] = position of the m-th set bit of the canonical mask bits,
// woff[w] = number of set bits in words [0, w)
__global__ void idx_count_kernel(const uint32_t* __restrict__ bits, int64_t nwords, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t red[32];
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kIdxWords;
  uint32_t c = 0;
  for (int i = threadIdx.x; i < kIdxWords; i += blockDim.x) {
    const int64_t w = w0 + i;
    if (w < nwords) c += __popc(bits[w]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFullA, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
    cnt[blockIdx.x] = t;
  }
}

// single block of 1024: exclusive scan of cnt[0..nb) -> off (uint64), total -> *mc
__global__ void __launch_bounds__(1024) idx_scan_kernel(const uint32_t* __restrict__ cnt, int nb,
                                                        uint64_t* __restrict__ off, uint64_t* __restrict__ mc) {
  __shared__ uint64_t carry;
  __shared__ uint64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const uint64_t v = i < nb ? cnt[i] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFullA, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint64_t s = wsum[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFullA, s, o);
        if (threadIdx.x >= o) s += y;
      }
      wsum[threadIdx.x] = s;  // inclusive over warps
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    const uint64_t excl = carry + (w > 0 ? wsum[w - 1] : 0) + x - v;
    if (i < nb) off[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *mc = carry;
}

// block b: words [b*kIdxWords, ...), one word per thread, block scan of the popcounts
__global__ void __launch_bounds__(kIdxWords) idx_write_kernel(const uint32_t* __restrict__ bits, int64_t nwords,
                                                              const uint64_t* __restrict__ off,
                                                              uint32_t* __restrict__ idx,
                                                              uint32_t* __restrict__ woff) {
  __shared__ uint32_t wsum[32];
  const int64_t w = static_cast<int64_t>(blockIdx.x) * kIdxWords + threadIdx.x;
  const uint32_t word = w < nwords ? bits[w] : 0u;
  const uint32_t c = __popc(word);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFullA, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t s = wsum[threadIdx.x];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullA, s, o);
      if (threadIdx.x >= o) s += y;
    }
    wsum[threadIdx.x] = s;
  }
  __syncthreads();
  const int wi = threadIdx.x >> 5;
  uint64_t pos = off[blockIdx.x] + (wi > 0 ? wsum[wi - 1] : 0) + x - c;
  if (w < nwords) woff[w] = static_cast<uint32_t>(pos);
  uint32_t rest = word;
  while (rest) {
    const int b = __ffs(rest) - 1;
    rest &= rest - 1;
    idx[pos++] = static_cast<uint32_t>(w * 32 + b);
  }
}

// row_off[r] = first compact index of code row r = k*Hc + u (r in [0, K*Hc]), from the sorted idx
__global__ void row_off_kernel(const uint32_t* __restrict__ idx, int64_t mc, int Wc, int64_t nrows,
                               uint64_t* __restrict__ row_off) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= mc) return;
  const int64_t row = idx[m] / Wc;
  const int64_t prev = m == 0 ? -1 : static_cast<int64_t>(idx[m - 1] / Wc);
  for (int64_t r = prev + 1; r <= row; ++r) row_off[r] = m;
  if (m == mc - 1)
    for (int64_t r = row + 1; r <= nrows; ++r) row_off[r] = mc;
}

// ---- A^T e on the selected codes (block (row band, n)):
//   c = sum_ab d[k,a,b] e[n, u-P+a, v-P+b];  out = sign*c (+ rho v, part += v*out, when v != null).
// A block takes kDtrBR code rows [u0, u0+BR) of every plane k: it stages the image rows
// [u0-P, u0+BR) (zero-padded to columns [-P, W+P), row pitch We = S mod 32 so that tap
// t = a*S + b of code (u, v) sits in bank (t + const) mod 32) in smem once for all K planes.
// A warp takes one plane k: the band's selected codes of plane k are one contiguous range of
// the compact list.  The S*S taps are spread over the 32 lanes (tap t = lane + 32 i, with its
// smem offset and d value in registers), so a code costs ceil(S*S/32) conflict-free smem loads
// + FMAs per lane; a batch of 32 codes is reduce-scattered over the warp (31 shuffles), leaving
// lane j with code j: coalesced stores, fp64 dot partials spread over lanes.
constexpr int kDtrBR = 4;

__host__ __device__ constexpr int dtr_pitch(int W, int P, int S) {
  // smallest pitch >= W + 2P with pitch = S (mod 32)
  return W + 2 * P + (((S - (W + 2 * P)) % 32) + 32) % 32;
}

template <int S>
__global__ void __launch_bounds__(kAT) masked_dtr_kernel(Geom g, const uint32_t* __restrict__ idx,
                                                         const uint64_t* __restrict__ row_off, int64_t ms,
                                                         const float* __restrict__ e, const float* __restrict__ d,
                                                         const float* __restrict__ v, float rho, float sign,
                                                         float* __restrict__ out, double* __restrict__ part) {
  constexpr int NT = (S * S + 31) / 32;  // taps per lane
  extern __shared__ float es[];          // [BR + S - 1][We]
  __shared__ double red[kAT / 32];
  const int u0 = blockIdx.x * kDtrBR, n = blockIdx.y;
  const int nrow = min(kDtrBR, g.Hc - u0);
  const int We = dtr_pitch(g.W, g.P, S);
  const int ER = kDtrBR + S - 1;
  {
    const float* en = e + static_cast<int64_t>(n) * g.H * g.W;
    for (int t = threadIdx.x; t < ER * We; t += kAT) {
      const int a = t / We, col = t - a * We;
      const int i = u0 - g.P + a, j = col - g.P;
      const bool in = i >= 0 && i < g.H && j >= 0 && j < g.W;
      es[t] = in ? __ldg(en + static_cast<int64_t>(i) * g.W + j) : 0.f;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int toff[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int t = lane + 32 * i;
    toff[i] = t < S * S ? (t / S) * We + (t % S) : 0;
  }
  double acc = 0.0;
  for (int k = wid; k < g.K; k += kAT / 32) {
    const int64_t rowi = static_cast<int64_t>(k) * g.Hc + u0;
    const int64_t m0 = static_cast<int64_t>(row_off[rowi]), m1 = static_cast<int64_t>(row_off[rowi + nrow]);
    if (m0 == m1) continue;
    float dt[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const int t = lane + 32 * i;
      dt[i] = t < S * S ? __ldg(d + static_cast<int64_t>(k) * S * S + t) : 0.f;
    }
    const uint32_t base = static_cast<uint32_t>(rowi * g.Wc);
    for (int64_t mb = m0; mb < m1; mb += 32) {
      const int nb = static_cast<int>(min(static_cast<int64_t>(32), m1 - mb));
      int myo = 0;
      if (lane < nb) {
        const uint32_t rel = __ldg(idx + mb + lane) - base;  // (u - u0) * Wc + v
        const uint32_t du = rel / g.Wc;
        myo = static_cast<int>(du * We + (rel - du * g.Wc));
      }
      float cs[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int o = __shfl_sync(kFullA, myo, i);
        float c = 0.f;
        if (i < nb) {
#pragma unroll
          for (int q = 0; q < NT; ++q) c = fmaf(dt[q], es[toff[q] + o], c);
        }
        cs[i] = c;
      }
      // reduce-scatter: lane j ends with the warp total of code j
#pragma unroll
      for (int o = 16, cnt = 32; o > 0; o >>= 1, cnt >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < cnt / 2; ++i) {
          const float send = hi ? cs[i] : cs[i + cnt / 2];
          const float keep = hi ? cs[i + cnt / 2] : cs[i];
          cs[i] = keep + __shfl_xor_sync(kFullA, send, o);
        }
      }
      if (lane < nb) {
        const int64_t gi = static_cast<int64_t>(n) * ms + mb + lane;
        const float c = cs[0];
        float o = sign * c;
        if (v != nullptr) {
          const float vi = v[gi];
          o = fmaf(rho, vi, o);
          acc += static_cast<double>(vi) * static_cast<double>(o);
        }
        out[gi] = o;
      }
    }
  }
  if (part != nullptr) {
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
  }
}

// A^T e from a dense correlation: out[n][m] = sign * Cd[n][idx[m]] (+ rho v, part += v*out,
// when v != null) -- Cd = D^T e at every position, written by the tensor-core code_h kernel in
// plain mode.  Thread per 4 consecutive m (4 independent gathers, float4 loads / stores over the
// padded stride; pads get 0).
__global__ void gather_kernel(Geom g, const uint32_t* __restrict__ idx, int64_t mc, int64_t ms,
                              const float* __restrict__ Cd, const float4* __restrict__ v, float rho, float sign,
                              float4* __restrict__ out, double* __restrict__ part) {
  __shared__ double red[kAT / 32];
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  const float* Cn = Cd + static_cast<int64_t>(n) * nc;
  const int64_t m4 = ms / 4;
  double acc = 0.0;
  // 4 grid-stride steps per batch with all their index -> value loads issued first (one dependent
  // latency per batch instead of per step); the dot partial keeps the per-thread ascending order
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kAT;
  for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; t0 < m4; t0 += 4 * stride) {
    float c[4][4];
    float4 vi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * stride;
      const int64_t m = 4 * t;
      if (m + 4 <= mc) {
        const uint4 l4 = __ldg(reinterpret_cast<const uint4*>(idx) + t);
        c[u][0] = Cn[l4.x]; c[u][1] = Cn[l4.y]; c[u][2] = Cn[l4.z]; c[u][3] = Cn[l4.w];
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) c[u][j] = m + j < mc ? Cn[__ldg(idx + m + j)] : 0.f;
      }
      vi[u] = (v != nullptr && t < m4) ? v[static_cast<int64_t>(n) * m4 + t] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * stride;
      if (t >= m4) break;
      const int64_t gi = static_cast<int64_t>(n) * m4 + t;
      float4 o = make_float4(sign * c[u][0], sign * c[u][1], sign * c[u][2], sign * c[u][3]);
      if (v != nullptr) {
        o.x = fmaf(rho, vi[u].x, o.x); o.y = fmaf(rho, vi[u].y, o.y); o.z = fmaf(rho, vi[u].z, o.z);
        o.w = fmaf(rho, vi[u].w, o.w);
        acc += static_cast<double>(vi[u].x) * o.x + static_cast<double>(vi[u].y) * o.y +
               static_cast<double>(vi[u].z) * o.z + static_cast<double>(vi[u].w) * o.w;
      }
      out[gi] = o;
    }
  }
  if (part != nullptr) {
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
  }
}

// W = Y = z[n][idx], U = 0  (pads of the [N][ms] vectors stay 0 from the per-call clear)
__global__ void admm_init_kernel(Geom g, const uint32_t* __restrict__ idx, int64_t mc, int64_t ms,
                                 const float* __restrict__ z, float* __restrict__ W, float* __restrict__ Y) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < mc;
       m += static_cast<int64_t>(gridDim.x) * kAT) {
    const int64_t gi = static_cast<int64_t>(n) * ms + m;
    const float zv = z[static_cast<int64_t>(n) * nc + __ldg(idx + m)];
    W[gi] = zv;
    Y[gi] = zv;
  }
}

// Dense expansion of a compact vector into the code buffer Zd, zeros off the mask.  A warp takes
// 32 consecutive mask words (1024 positions): lane j loads word/offset j (coalesced), then for each
// word the lanes write its 32 positions (one 128-B line) with the selected lanes reading their
// consecutive compact entries; 8 words per round are unrolled so 8 loads per lane are in flight.
// With PV != null the CG direction is formed on the way: PV = R + beta PV (beta = rr_new / rr per
// image, 0 when rr == 0; PV = R when rr == null) and Zd gets PV; otherwise Zd gets R.
// max|written| -> atomicMax(bound).
__global__ void __launch_bounds__(256) expand_kernel(int64_t nper, const uint32_t* __restrict__ bits,
                                                     const uint32_t* __restrict__ woff, int64_t ms,
                                                     const float* __restrict__ R, float* __restrict__ PV,
                                                     const double* __restrict__ rr,
                                                     const double* __restrict__ rr_new, float* __restrict__ Zd,
                                                     uint32_t* __restrict__ bound) {
  const int n = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const bool dir = rr != nullptr;
  float beta = 0.f;
  if (dir) {
    const double r0 = rr[n], r1 = rr_new[n];
    beta = r0 > 0.0 ? static_cast<float>(r1 / r0) : 0.f;
  }
  const float* Rn = R + static_cast<int64_t>(n) * ms;
  float* PVn = PV != nullptr ? PV + static_cast<int64_t>(n) * ms : nullptr;
  float* Zn = Zd + static_cast<int64_t>(n) * nper;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t mx = 0u;
  const int64_t nwords = (nper + 31) / 32;
  const int64_t nchunk = (nwords + 31) / 32;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunk;
       ch += wstride) {
    const int64_t w0 = ch * 32;
    const bool wok = w0 + lane < nwords;
    const uint32_t myword = wok ? __ldg(bits + w0 + lane) : 0u;
    const uint32_t myoff = wok ? __ldg(woff + w0 + lane) : 0u;
#pragma unroll 1
    for (int i0 = 0; i0 < 32; i0 += 8) {
      // all compact loads of the round before any PV store (the stores alias PV for the
      // compiler, so interleaving them would serialise the loads)
      float val[8], pv[8];
      uint32_t mi[8];
      bool on[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t word = __shfl_sync(kFullA, myword, i0 + i);
        const uint32_t off = __shfl_sync(kFullA, myoff, i0 + i);
        on[i] = (word >> lane) & 1u;
        mi[i] = off + __popc(word & lt);
        val[i] = on[i] ? Rn[mi[i]] : 0.f;
        pv[i] = (on[i] && dir) ? PVn[mi[i]] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (dir) val[i] = fmaf(beta, pv[i], val[i]);
        if (on[i] && PVn != nullptr) PVn[mi[i]] = val[i];
        if (!on[i]) val[i] = 0.f;
        mx = max(mx, __float_as_uint(fabsf(val[i])));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t pos = (w0 + i0 + i) * 32 + lane;
        if (pos < nper) Zn[pos] = val[i];
      }
    }
  }
  block_atomic_max(mx, bound);
}

// expand_kernel for nper % 4 == 0 (every image row of Zd 16-B aligned), staged through shared
// memory.  A block takes a span of kExpWords = 256 mask words (8192 positions, one word per
// thread); the span's selected codes are one contiguous compact segment [woff[w0], woff[w0] + cnt),
// which the block reads with coalesced loads (forming PV on the way) into smem, then each warp
// writes its 32 words (1024 positions) as float4 lines: in round j (0..7) lane L owns positions
// 128 j + 4 L .. +3, nibble L & 7 of the warp's word 4 j + (L >> 3).  Every load of a span is
// independent of the others, so a block keeps ~cnt / 256 loads per thread in flight instead of a
// chain of dependent word -> value loads per warp.
constexpr int kExpWords = 256;
__global__ void __launch_bounds__(kExpWords) expand_seg_kernel(int64_t nper, const uint32_t* __restrict__ bits,
                                                               const uint32_t* __restrict__ woff, int64_t ms,
                                                               const float* __restrict__ R, float* __restrict__ PV,
                                                               const double* __restrict__ rr,
                                                               const double* __restrict__ rr_new,
                                                               float* __restrict__ Zd, uint32_t* __restrict__ bound) {
  __shared__ float seg[kExpWords * 32];
  __shared__ uint32_t span[2];
  const int n = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool dir = rr != nullptr;
  float beta = 0.f;
  if (dir) {
    const double r0 = rr[n], r1 = rr_new[n];
    beta = r0 > 0.0 ? static_cast<float>(r1 / r0) : 0.f;
  }
  const float* Rn = R + static_cast<int64_t>(n) * ms;
  float* PVn = PV != nullptr ? PV + static_cast<int64_t>(n) * ms : nullptr;
  float4* Zn = reinterpret_cast<float4*>(Zd + static_cast<int64_t>(n) * nper);
  const int sh = 4 * (lane & 7);
  const uint32_t below = (1u << sh) - 1u;
  uint32_t mx = 0u;
  const int64_t nwords = (nper + 31) / 32;
  const int64_t wstep = static_cast<int64_t>(gridDim.x) * kExpWords;
  int64_t wn = static_cast<int64_t>(blockIdx.x) * kExpWords + threadIdx.x;
  uint32_t nword = wn < nwords ? __ldg(bits + wn) : 0u;  // the next span's word / offset, one span ahead
  uint32_t noff = wn < nwords ? __ldg(woff + wn) : 0u;
  for (int64_t w0 = static_cast<int64_t>(blockIdx.x) * kExpWords; w0 < nwords; w0 += wstep) {
    const int64_t w = w0 + threadIdx.x;
    const uint32_t myword = nword, myoff = noff;
    wn = w + wstep;
    nword = wn < nwords ? __ldg(bits + wn) : 0u;
    noff = wn < nwords ? __ldg(woff + wn) : 0u;
    if (threadIdx.x == 0) span[0] = myoff;
    // the last word of the span (or of the mask) closes the segment
    if (w < nwords && (threadIdx.x == kExpWords - 1 || w == nwords - 1)) span[1] = myoff + __popc(myword);
    __syncthreads();
    const uint32_t mb = span[0];
    const int cnt = static_cast<int>(span[1] - mb);
    // batches of 4 per thread, every load of a batch before its PV stores (which alias PV for the
    // compiler and would otherwise serialise the loads)
    for (int i0 = threadIdx.x; i0 < cnt; i0 += 4 * kExpWords) {
      float rv[4], pv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kExpWords;
        rv[u] = i < cnt ? Rn[mb + i] : 0.f;
        pv[u] = (i < cnt && dir) ? PVn[mb + i] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kExpWords;
        if (i < cnt) {
          float x = rv[u];
          if (dir) x = fmaf(beta, pv[u], x);
          if (PVn != nullptr) PVn[mb + i] = x;
          seg[i] = x;
          mx = max(mx, __float_as_uint(fabsf(x)));
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int src = 4 * j + (lane >> 3);
      const uint32_t word = __shfl_sync(kFullA, myword, src);
      const uint32_t off = __shfl_sync(kFullA, myoff, src) - mb;
      const uint32_t nib = (word >> sh) & 0xFu;
      uint32_t m = off + __popc(word & below);
      float v[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const bool on = (nib >> b) & 1u;
        v[b] = on ? seg[m] : 0.f;
        m += on ? 1u : 0u;
      }
      const int64_t pos = (w0 + 32 * warp) * 32 + 128 * j + 4 * lane;
      if (pos < nper) Zn[pos / 4] = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();
  }
  block_atomic_max(mx, bound);
}

// z[n][idx[m]] = Y[n][m] (selected positions only); max|written| -> atomicMax(bound)
__global__ void scatter_kernel(Geom g, const uint32_t* __restrict__ idx, int64_t mc, int64_t ms,
                               const float* __restrict__ Y, float* __restrict__ z, uint32_t* __restrict__ bound) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  uint32_t mx = 0u;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < mc;
       m += static_cast<int64_t>(gridDim.x) * kAT) {
    const float val = Y[static_cast<int64_t>(n) * ms + m];
    z[static_cast<int64_t>(n) * nc + __ldg(idx + m)] = val;
    mx = max(mx, __float_as_uint(fabsf(val)));
  }
  block_atomic_max(mx, bound);
}

__device__ __forceinline__ double dot4(float4 a) {
  return static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y + static_cast<double>(a.z) * a.z +
         static_cast<double>(a.w) * a.w;
}

// Explicit CG residual (the oracle's order): R = ATB + rho (Y - U) - Q, part = sum R^2.
// With init != 0 it instead forms ATB = R + Q - rho Y from R = A^T b - A^T A w0 (Y = W = w0).
__global__ void cg_resid_kernel(int64_t ms, float4* __restrict__ ATB, const float4* __restrict__ Y,
                                const float4* __restrict__ U, const float4* __restrict__ Q, float rho,
                                float4* __restrict__ R, double* __restrict__ part, int init) {
  __shared__ double red[kAT / 32];
  const int n = blockIdx.y;
  const int64_t m4 = ms / 4;
  double acc = 0.0;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < m4;
       m += static_cast<int64_t>(gridDim.x) * kAT) {
    const int64_t gi = static_cast<int64_t>(n) * m4 + m;
    const float4 y = Y[gi], q = Q[gi];
    if (init) {
      const float4 r = R[gi];
      ATB[gi] = make_float4(r.x + q.x - rho * y.x, r.y + q.y - rho * y.y, r.z + q.z - rho * y.z,
                            r.w + q.w - rho * y.w);
      acc += dot4(r);
    } else {
      const float4 a = ATB[gi], uu = U[gi];
      float4 r;
      r.x = a.x + rho * (y.x - uu.x) - q.x;
      r.y = a.y + rho * (y.y - uu.y) - q.y;
      r.z = a.z + rho * (y.z - uu.z) - q.z;
      r.w = a.w + rho * (y.w - uu.w) - q.w;
      R[gi] = r;
      acc += dot4(r);
    }
  }
  const double t = block_sum_d(acc, red);
  if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

// per image (one warp each): out[n] = sum_b part[n][b]
__global__ void image_sum_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double slot;
  const double s = image_total(part, blockIdx.x, nb, &slot);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// CG step: pq = sum_b part_pq[n][b]; a = rr / pq (0 if rr == 0 or pq <= 0); W += a PV,
// R -= a Q; part_rr = sum R^2
__global__ void cg_step_kernel(int64_t ms, const double* __restrict__ rr, const double* __restrict__ part_pq,
                               int nb_pq, float4* __restrict__ W, float4* __restrict__ R,
                               const float4* __restrict__ PV, const float4* __restrict__ Q,
                               double* __restrict__ part_rr) {
  __shared__ double red[kAT / 32];
  __shared__ double slot;
  const int n = blockIdx.y;
  const double d0 = image_total(part_pq, n, nb_pq, &slot);
  const double r0 = rr[n];
  const float a = (r0 > 0.0 && d0 > 0.0) ? static_cast<float>(r0 / d0) : 0.f;
  const int64_t m4 = ms / 4;
  double acc = 0.0;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < m4;
       m += static_cast<int64_t>(gridDim.x) * kAT) {
    const int64_t gi = static_cast<int64_t>(n) * m4 + m;
    float4 w = W[gi], r = R[gi];
    const float4 pv = PV[gi], q = Q[gi];
    w.x = fmaf(a, pv.x, w.x); w.y = fmaf(a, pv.y, w.y); w.z = fmaf(a, pv.z, w.z); w.w = fmaf(a, pv.w, w.w);
    r.x = fmaf(-a, q.x, r.x); r.y = fmaf(-a, q.y, r.y); r.z = fmaf(-a, q.z, r.z); r.w = fmaf(-a, q.w, r.w);
    W[gi] = w;
    R[gi] = r;
    acc += dot4(r);
  }
  const double t = block_sum_d(acc, red);
  if (threadIdx.x == 0) part_rr[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

// One ADMM update on a float lane, carrying the CG residual to the new right-hand side:
//   w^ = alpha w + (1 - alpha) y;  y' = S(w^ + u, kappa);  u' = u + w^ - y';
//   r += rho ((y' - u') - (y - u))   [r = ATB + rho (y - u) - (A^T A + rho I) w]
__device__ __forceinline__ void admm_upd1(float w, float& y, float& u, float& r, float alpha, float kappa, float rho) {
  const float wh = fmaf(alpha, w, (1.f - alpha) * y);
  const float q = wh + u;
  const float yn = q > kappa ? q - kappa : (q < -kappa ? q + kappa : 0.f);
  const float un = u + (wh - yn);
  r = fmaf(rho, (yn - un) - (y - u), r);
  u = un;
  y = yn;
}

__global__ void admm_update_kernel(int64_t ms, const float4* __restrict__ W, float4* __restrict__ Y,
                                   float4* __restrict__ U, float4* __restrict__ R, float alpha, float kappa, float rho,
                                   double* __restrict__ part) {
  __shared__ double red[kAT / 32];
  const int n = blockIdx.y;
  const int64_t m4 = ms / 4;
  double acc = 0.0;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < m4;
       m += static_cast<int64_t>(gridDim.x) * kAT) {
    const int64_t gi = static_cast<int64_t>(n) * m4 + m;
    const float4 w = W[gi];
    float4 y = Y[gi], uu = U[gi], r = R[gi];
    admm_upd1(w.x, y.x, uu.x, r.x, alpha, kappa, rho);
    admm_upd1(w.y, y.y, uu.y, r.y, alpha, kappa, rho);
    admm_upd1(w.z, y.z, uu.z, r.z, alpha, kappa, rho);
    admm_upd1(w.w, y.w, uu.w, r.w, alpha, kappa, rho);
    Y[gi] = y;
    U[gi] = uu;
    R[gi] = r;
    acc += dot4(r);
  }
  const double t = block_sum_d(acc, red);
  if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

// part = per-block sum R^2
__global__ void sumsq_kernel(int64_t ms, const float4* __restrict__ R, double* __restrict__ part) {
  __shared__ double red[kAT / 32];
  const int n = blockIdx.y;
  const int64_t m4 = ms / 4;
  double acc = 0.0;
  for (int64_t m = static_cast<int64_t>(blockIdx.x) * kAT + threadIdx.x; m < m4;
       m += static_cast<int64_t>(gridDim.x) * kAT)
    acc += dot4(R[static_cast<int64_t>(n) * m4 + m]);
  const double t = block_sum_d(acc, red);
  if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

}  // namespace

int admm_blocks(const Geom& g, int64_t ms) {
  const int n = g.N > 0 ? g.N : 1;
  int64_t nb = (ms / 4 + kAT * 2 - 1) / (kAT * 2);
  const int64_t cap = (148 * 16 + n - 1) / n;
  if (nb > cap) nb = cap;
  if (nb < 1) nb = 1;
  return static_cast<int>(nb);
}

int admm_idx_blocks(const Geom& g) {
  const int64_t nwords = (static_cast<int64_t>(g.K) * g.Hc * g.Wc + 31) / 32;
  return static_cast<int>((nwords + kIdxWords - 1) / kIdxWords);
}

cudaError_t launch_admm_index(const Geom& g, const uint32_t* bits, uint32_t* cnt, uint64_t* off, uint64_t* mc,
                              uint32_t* idx, uint32_t* woff, cudaStream_t st) {
  const int64_t nwords = (static_cast<int64_t>(g.K) * g.Hc * g.Wc + 31) / 32;
  const int nb = admm_idx_blocks(g);
  idx_count_kernel<<<nb, 256, 0, st>>>(bits, nwords, cnt);
  idx_scan_kernel<<<1, 1024, 0, st>>>(cnt, nb, off, mc);
  idx_write_kernel<<<nb, kIdxWords, 0, st>>>(bits, nwords, off, idx, woff);
  return cudaGetLastError();
}

cudaError_t launch_admm_row_off(const Geom& g, const uint32_t* idx, int64_t mc, uint64_t* row_off,
                                cudaStream_t st) {
  if (mc <= 0) return cudaSuccess;
  row_off_kernel<<<static_cast<unsigned>((mc + 255) / 256), 256, 0, st>>>(idx, mc, g.Wc,
                                                                          static_cast<int64_t>(g.K) * g.Hc, row_off);
  return cudaGetLastError();
}

int admm_dtr_blocks(const Geom& g) { return (g.Hc + kDtrBR - 1) / kDtrBR; }

template <int S>
static cudaError_t run_dtr(const Geom& g, const uint32_t* idx, const uint64_t* row_off, int64_t ms, const float* e,
                           const float* d, const float* v, float rho, float sign, float* out, double* part,
                           cudaStream_t st) {
  const size_t smem = sizeof(float) * (kDtrBR + S - 1) * dtr_pitch(g.W, g.P, S);
  if (smem > 48 * 1024) {
    cudaError_t er = cudaFuncSetAttribute(masked_dtr_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem));
    if (er != cudaSuccess) return er;
  }
  masked_dtr_kernel<S><<<dim3(admm_dtr_blocks(g), g.N), kAT, smem, st>>>(g, idx, row_off, ms, e, d, v, rho, sign, out,
                                                                         part);
  return cudaGetLastError();
}

cudaError_t launch_masked_dtr(const Geom& g, const uint32_t* idx, const uint64_t* row_off, int64_t ms, const float* e,
                              const float* d, const float* v, float rho, float sign, float* out, double* part,
                              cudaStream_t st) {
  switch (g.S) {
    case 1: return run_dtr<1>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    case 3: return run_dtr<3>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    case 5: return run_dtr<5>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    case 7: return run_dtr<7>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    case 9: return run_dtr<9>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    case 11: return run_dtr<11>(g, idx, row_off, ms, e, d, v, rho, sign, out, part, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_admm_gather(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* Cd,
                               const float* v, float rho, float sign, float* out, double* part, cudaStream_t st) {
  gather_kernel<<<dim3(admm_blocks(g, ms), g.N), kAT, 0, st>>>(g, idx, mc, ms, Cd, reinterpret_cast<const float4*>(v),
                                                                rho, sign, reinterpret_cast<float4*>(out), part);
  return cudaGetLastError();
}

cudaError_t launch_admm_init(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* z, float* W,
                             float* Y, cudaStream_t st) {
  admm_init_kernel<<<dim3(admm_blocks(g, ms), g.N), kAT, 0, st>>>(g, idx, mc, ms, z, W, Y);
  return cudaGetLastError();
}

cudaError_t launch_admm_expand(const Geom& g, const uint32_t* bits, const uint32_t* woff, int64_t ms, const float* R,
                               float* PV, const double* rr, const double* rr_new, float* Zd, uint32_t* bound,
                               cudaStream_t st) {
  const int64_t nper = static_cast<int64_t>(g.K) * g.Hc * g.Wc;
  const int64_t nchunk = ((nper + 31) / 32 + 31) / 32;
  int64_t nb = (nchunk + 7) / 8;  // 8 warps per block
  const int64_t cap = (148 * 16 + g.N - 1) / g.N;
  if (nb > cap) nb = cap;
  const char* ev = std::getenv("CSC_ADMM_EXPAND");
  const bool scalar = ev != nullptr && std::strcmp(ev, "scalar") == 0;
  if (nper % 4 == 0 && (reinterpret_cast<uintptr_t>(Zd) & 15u) == 0 && !scalar) {
    int64_t nbs = ((nper + 31) / 32 + kExpWords - 1) / kExpWords;
    const int64_t caps = (148 * 6 + g.N - 1) / g.N;  // ~6 resident blocks per SM (33 KB smem each)
    if (nbs > caps) nbs = caps;
    expand_seg_kernel<<<dim3(static_cast<unsigned>(nbs), g.N), kExpWords, 0, st>>>(nper, bits, woff, ms, R, PV, rr,
                                                                                   rr_new, Zd, bound);
  } else
    expand_kernel<<<dim3(static_cast<unsigned>(nb), g.N), 256, 0, st>>>(nper, bits, woff, ms, R, PV, rr, rr_new, Zd,
                                                                         bound);
  return cudaGetLastError();
}

cudaError_t launch_admm_scatter(const Geom& g, const uint32_t* idx, int64_t mc, int64_t ms, const float* Y, float* z,
                                uint32_t* bound, cudaStream_t st) {
  scatter_kernel<<<dim3(admm_blocks(g, ms), g.N), kAT, 0, st>>>(g, idx, mc, ms, Y, z, bound);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const Geom& g, int64_t ms, const float* R, double* part, double* rr, cudaStream_t st) {
  const int nb = admm_blocks(g, ms);
  sumsq_kernel<<<dim3(nb, g.N), kAT, 0, st>>>(ms, reinterpret_cast<const float4*>(R), part);
  image_sum_kernel<<<g.N, 32, 0, st>>>(part, nb, rr);
  return cudaGetLastError();
}

cudaError_t launch_cg_resid(const Geom& g, int64_t ms, float* ATB, const float* Y, const float* U, const float* Q,
                            float rho, float* R, double* part, double* rr, bool init, cudaStream_t st) {
  const int nb = admm_blocks(g, ms);
  cg_resid_kernel<<<dim3(nb, g.N), kAT, 0, st>>>(ms, reinterpret_cast<float4*>(ATB), reinterpret_cast<const float4*>(Y),
                                                 reinterpret_cast<const float4*>(U), reinterpret_cast<const float4*>(Q),
                                                 rho, reinterpret_cast<float4*>(R), part, init ? 1 : 0);
  image_sum_kernel<<<g.N, 32, 0, st>>>(part, nb, rr);
  return cudaGetLastError();
}

cudaError_t launch_cg_step(const Geom& g, int64_t ms, const double* rr, const double* part_pq, int nb_pq, float* W,
                           float* R,
                           const float* PV, const float* Q, double* part_rr, double* rr_new, cudaStream_t st) {
  const int nb = admm_blocks(g, ms);
  cg_step_kernel<<<dim3(nb, g.N), kAT, 0, st>>>(ms, rr, part_pq, nb_pq, reinterpret_cast<float4*>(W),
                                                reinterpret_cast<float4*>(R), reinterpret_cast<const float4*>(PV),
                                                reinterpret_cast<const float4*>(Q), part_rr);
  image_sum_kernel<<<g.N, 32, 0, st>>>(part_rr, nb, rr_new);
  return cudaGetLastError();
}

cudaError_t launch_admm_update(const Geom& g, int64_t ms, const float* W, float* Y, float* U, float* R, float alpha,
                               float kappa, float rho, double* part, double* rr, cudaStream_t st) {
  const int nb = admm_blocks(g, ms);
  admm_update_kernel<<<dim3(nb, g.N), kAT, 0, st>>>(ms, reinterpret_cast<const float4*>(W),
                                                    reinterpret_cast<float4*>(Y), reinterpret_cast<float4*>(U),
                                                    reinterpret_cast<float4*>(R), alpha, kappa, rho, part);
  image_sum_kernel<<<g.N, 32, 0, st>>>(part, nb, rr);
  return cudaGetLastError();
}

}  // namespace csc

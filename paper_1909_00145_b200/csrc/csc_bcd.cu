// csc_bcd.cu -- projected block-coordinate descent on the filters (PAPER.md
// P:313-317 "solved by projected block coordinate decent ... a single iteration is enough with f
// computed in previous iteration as a warm start", readings B1-B4).  The sweep itself
// is driven by csc_api.cu (csc_filter_step_bcd):
//   once per sweep:  C_kk = sum_n Z_nk^T Z_nk for every k (bcd_gram_kernel, fp64), then
//                    A_k^-1 = (C_kk + eps tr(C_kk)/M I)^-1 via Cholesky (bcd_inverse_kernel)
//   per filter k:    g_k = sum_n Z_nk^T r_n (bcd_gk_kernel, fp64, current residual)
//                    d_k <- P_ball(d_k - A_k^-1 g_k), delta = d_k,new - d_k,old (bcd_update_kernel)
//                    r <- r + Z_k delta (bcd_resid_kernel)
// All sums in fp64 in a fixed order (deterministic).  The products of fp32 codes are exact in fp64.
#include "csc_internal.cuh"

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace csc {
namespace {

constexpr unsigned kFullB = 0xffffffffu;
constexpr int kGramThreads = 256;
constexpr int kGramBR = 8;  // output rows per staged band

// ---- Gram blocks: block (split, k) accumulates sum over its images n and all positions of
// X[p][t] X[p][t'] for the 4x4 tap tiles (T1 <= T2) its threads own; X[p][t] = z[n,k,i+P-a,j+P-b].
__global__ void __launch_bounds__(kGramThreads) bcd_gram_kernel(Geom g, const float* __restrict__ z, int nsplit,
                                                                double* __restrict__ gpart) {
  extern __shared__ double zs[];  // [kGramBR + P][Wc] + 1 zero, staged as fp64 (exact)
  const int k = blockIdx.y, sp = blockIdx.x;
  const int M = g.S * g.S;
  const int NT = (M + 3) / 4;                // tap tiles per dimension
  const int ntiles = NT * (NT + 1) / 2;      // upper-triangular tile pairs
  const int rows = kGramBR + g.P;
  const int zero_at = rows * g.Wc;
  // this thread's (up to 2) tile pairs and their smem tap offsets
  int off1[2][4], off2[2][4];
  bool own[2];
  for (int q = 0; q < 2; ++q) {
    int id = threadIdx.x + q * kGramThreads;
    own[q] = id < ntiles;
    int T1 = 0;
    if (own[q]) {
      while (id >= NT - T1) {
        id -= NT - T1;
        ++T1;
      }
    }
    const int T2 = T1 + (own[q] ? id : 0);
    for (int e = 0; e < 4; ++e) {
      const int t1 = 4 * T1 + e, t2 = 4 * T2 + e;
      off1[q][e] = t1 < M ? (g.P - t1 / g.S) * g.Wc + (g.P - t1 % g.S) : -1;
      off2[q][e] = t2 < M ? (g.P - t2 / g.S) * g.Wc + (g.P - t2 % g.S) : -1;
    }
  }
  double acc[2][4][4];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[q][a][b] = 0.0;
  const int n0 = static_cast<int>((static_cast<int64_t>(sp) * g.N) / nsplit);
  const int n1 = static_cast<int>((static_cast<int64_t>(sp + 1) * g.N) / nsplit);
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  if (threadIdx.x == 0) zs[zero_at] = 0.0;
  for (int n = n0; n < n1; ++n) {
    const float* zk = z + (static_cast<int64_t>(n) * g.K + k) * plane;
    for (int i0 = 0; i0 < g.H; i0 += kGramBR) {
      __syncthreads();
      const int nr = min(rows, g.Hc - i0);
      for (int e = threadIdx.x; e < rows * g.Wc; e += kGramThreads) {
        const int rr = e / g.Wc;
        zs[e] = rr < nr ? static_cast<double>(__ldg(zk + static_cast<int64_t>(i0) * g.Wc + e)) : 0.0;
      }
      __syncthreads();
      const int ib = min(kGramBR, g.H - i0);
      for (int ii = 0; ii < ib; ++ii)
        for (int j = 0; j < g.W; ++j) {
          const int base = ii * g.Wc + j;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!own[q]) continue;
            double x1[4], x2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              x1[e] = zs[off1[q][e] >= 0 ? base + off1[q][e] : zero_at];
              x2[e] = zs[off2[q][e] >= 0 ? base + off2[q][e] : zero_at];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[q][a][b] = fma(x1[a], x2[b], acc[q][a][b]);
          }
        }
    }
  }
  // partial [k][sp][M][M] (the owned upper tiles; bcd_inverse_kernel mirrors them)
  double* out = gpart + (static_cast<int64_t>(k) * nsplit + sp) * M * M;
  for (int q = 0; q < 2; ++q) {
    if (!own[q]) continue;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        if (off1[q][a] < 0 || off2[q][b] < 0) continue;
        // recover t1, t2 from the offsets' tile ids
        int id = threadIdx.x + q * kGramThreads, T1 = 0;
        while (id >= NT - T1) {
          id -= NT - T1;
          ++T1;
        }
        const int t1 = 4 * T1 + a, t2 = 4 * (T1 + id) + b;
        out[static_cast<int64_t>(t1) * M + t2] = acc[q][a][b];
      }
  }
}

// ---- one block per k: C = sum of the partials (fixed order, upper tiles mirrored), tr, ridge,
// Cholesky, and the inverse A^-1 (column by column); flags[k] = 1 when tr(C) == 0 or a pivot fails.
__global__ void bcd_inverse_kernel(Geom g, const double* __restrict__ gpart, int nsplit, double ridge_rel,
                                   double* __restrict__ ainv, uint8_t* __restrict__ flags) {
  extern __shared__ double A[];  // [M][M]
  __shared__ int bad;
  const int k = blockIdx.x;
  const int M = g.S * g.S;
  const int NT = (M + 3) / 4;
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int t1 = e / M, t2 = e - t1 * M;
    // the owned entry is the one in the upper tile (T1 <= T2); within a diagonal tile both halves exist
    const int T1 = t1 / 4, T2 = t2 / 4;
    const int r1 = T1 <= T2 ? t1 : t2, r2 = T1 <= T2 ? t2 : t1;
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += gpart[(static_cast<int64_t>(k) * nsplit + sp) * M * M + static_cast<int64_t>(r1) * M + r2];
    A[e] = s;
  }
  (void)NT;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int m = 0; m < M; ++m) tr += A[m * M + m];
    if (!(tr > 0.0)) bad = 1;
    else {
      const double rd = ridge_rel * tr / static_cast<double>(M);
      for (int m = 0; m < M; ++m) A[m * M + m] += rd;
    }
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) flags[k] = 1;
    return;
  }
  // Cholesky in place (lower triangle), column by column
  for (int j = 0; j < M; ++j) {
    if (threadIdx.x == 0) {
      double s = A[j * M + j];
      for (int q = 0; q < j; ++q) s -= A[j * M + q] * A[j * M + q];
      if (!(s > 0.0)) bad = 1;
      A[j * M + j] = s > 0.0 ? sqrt(s) : 1.0;
    }
    __syncthreads();
    const double ljj = A[j * M + j];
    for (int i = j + 1 + threadIdx.x; i < M; i += blockDim.x) {
      double t = A[i * M + j];
      for (int q = 0; q < j; ++q) t -= A[i * M + q] * A[j * M + q];
      A[i * M + j] = t / ljj;
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) flags[k] = 1;
    return;
  }
  if (threadIdx.x == 0) flags[k] = 0;
  // A^-1 column c: L y = e_c, L^T x = y (one thread per column)
  double* out = ainv + static_cast<int64_t>(k) * M * M;
  for (int c = threadIdx.x; c < M; c += blockDim.x) {
    double y[128];
    for (int i = 0; i < M; ++i) {
      double t = i == c ? 1.0 : 0.0;
      for (int q = 0; q < i; ++q) t -= A[i * M + q] * y[q];
      y[i] = t / A[i * M + i];
    }
    for (int i = M - 1; i >= 0; --i) {
      double t = y[i];
      for (int q = i + 1; q < M; ++q) t -= A[q * M + i] * y[q];
      y[i] = t / A[i * M + i];
    }
    for (int i = 0; i < M; ++i) out[static_cast<int64_t>(i) * M + c] = y[i];
  }
}

// ---- g_k partials: block (n, row band) computes sum over its positions of r[p] X[p][t], t = tap
// (thread t < M), in fp64 -> part[blk][M]
constexpr int kGkBR = 6;
__global__ void bcd_gk_kernel(Geom g, int k, const float* __restrict__ z, const float* __restrict__ r,
                              double* __restrict__ part) {
  extern __shared__ double smd[];  // z rows [kGkBR + P][Wc], r rows [kGkBR][W], staged as fp64 (exact)
  const int nbands = (g.H + kGkBR - 1) / kGkBR;
  const int n = blockIdx.x / nbands, band = blockIdx.x - n * nbands;
  const int i0 = band * kGkBR;
  const int ib = min(kGkBR, g.H - i0);
  const int rows = kGkBR + g.P;
  double* zs = smd;
  double* rsm = smd + rows * g.Wc;
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  const float* zk = z + (static_cast<int64_t>(n) * g.K + k) * plane;
  for (int e = threadIdx.x; e < rows * g.Wc; e += blockDim.x) {
    const int rr = e / g.Wc;
    zs[e] = (i0 + rr < g.Hc) ? static_cast<double>(__ldg(zk + static_cast<int64_t>(i0) * g.Wc + e)) : 0.0;
  }
  for (int e = threadIdx.x; e < ib * g.W; e += blockDim.x)
    rsm[e] = static_cast<double>(r[(static_cast<int64_t>(n) * g.H + i0) * g.W + e]);
  __syncthreads();
  const int M = g.S * g.S;
  const int t = threadIdx.x;
  if (t < M) {
    const int a = t / g.S, b = t - a * g.S;
    double acc = 0.0;
    for (int ii = 0; ii < ib; ++ii) {
      const double* zrow = zs + (ii + g.P - a) * g.Wc + (g.P - b);
      const double* rrow = rsm + ii * g.W;
      double s0 = 0.0, s1 = 0.0;  // two chains against the fp64 FMA latency
      int j = 0;
      for (; j + 1 < g.W; j += 2) {
        s0 = fma(rrow[j], zrow[j], s0);
        s1 = fma(rrow[j + 1], zrow[j + 1], s1);
      }
      if (j < g.W) s0 = fma(rrow[j], zrow[j], s0);
      acc += s0 + s1;
    }
    part[static_cast<int64_t>(blockIdx.x) * M + t] = acc;
  }
}

// ---- gk[t] = sum of the g_k partials: one warp per tap, lane-strided partial sums then a fixed
// butterfly (deterministic)
__global__ void bcd_gsum_kernel(int M, const double* __restrict__ part, int nparts, double* __restrict__ gk) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= M) return;
  double s = 0.0;
  for (int b = lane; b < nparts; b += 32) s += part[static_cast<int64_t>(b) * M + t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullB, s, o);
  if (lane == 0) gk[t] = s;
}

// ---- one block: delta = -A^-1 g_k, e = d_k + delta, d_k <- e / max(1, ||e||) (fp32),
// dl = d_k,new - d_k,old (fp64).  Flagged filters: dl = 0, d_k unchanged.
__global__ void bcd_update_kernel(Geom g, int k, const double* __restrict__ gk, const double* __restrict__ ainv,
                                  const uint8_t* __restrict__ flags, float* __restrict__ d, double* __restrict__ dl) {
  __shared__ double gs[128], es[128], red[32];
  const int M = g.S * g.S;
  const int t = threadIdx.x;
  if (flags[k]) {
    if (t < M) dl[t] = 0.0;
    return;
  }
  if (t < M) gs[t] = gk[t];
  __syncthreads();
  double e = 0.0;
  if (t < M) {
    const double* row = ainv + (static_cast<int64_t>(k) * M + t) * M;
    double s = 0.0;
    for (int q = 0; q < M; ++q) s = fma(row[q], gs[q], s);
    e = static_cast<double>(d[static_cast<int64_t>(k) * M + t]) - s;
    es[t] = e;
  }
  double v = t < M ? e * e : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullB, v, o);
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  if (t == 0) {
    double nrm2 = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) nrm2 += red[w];
    red[0] = fmax(1.0, sqrt(nrm2));
  }
  __syncthreads();
  if (t < M) {
    const float dn = static_cast<float>(es[t] / red[0]);
    const int64_t di = static_cast<int64_t>(k) * M + t;
    dl[t] = static_cast<double>(dn) - static_cast<double>(d[di]);
    d[di] = dn;
  }
}

// ---- r[n,i,j] += sum_ab dl[a,b] z[n,k,i+P-a,j+P-b]  (fp32: r is fp32 and the update is small)
__global__ void bcd_resid_kernel(Geom g, int k, const float* __restrict__ z, const double* __restrict__ dl,
                                 float* __restrict__ r) {
  __shared__ float dls[128];
  const int M = g.S * g.S;
  if (threadIdx.x < M) dls[threadIdx.x] = static_cast<float>(dl[threadIdx.x]);
  __syncthreads();
  const int64_t npx = static_cast<int64_t>(g.N) * g.H * g.W;
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < npx;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = q / (static_cast<int64_t>(g.H) * g.W);
    const int64_t rem = q - n * g.H * g.W;
    const int i = static_cast<int>(rem / g.W), j = static_cast<int>(rem - static_cast<int64_t>(i) * g.W);
    const float* zk = z + (n * g.K + k) * plane;
    float s = 0.f;
    for (int a = 0; a < g.S; ++a)
      for (int b = 0; b < g.S; ++b)
        s = fmaf(dls[a * g.S + b], __ldg(zk + static_cast<int64_t>(i + g.P - a) * g.Wc + j + g.P - b), s);
    r[q] += s;
  }
}

// ---- Lag-structured Gram (the default when H, W > P): C_kk[(a,b),(a',b')] is the sum of
// Pi(u,v) = z[u,v] z[u+du, v+dv], du = a - a', dv = b - b', over the box [P-a, P-a+H) x
// [P-b, P-b+W) of the code plane -- a window of the plane's autocorrelation at lag (du, dv).  One
// thread per lag accumulates the 2D prefix sums Q(r, c) = sum_{u<r, v<c} Pi at the 2S row cuts
// {0..P} u {H..H+P} and the 2S column cuts {0..P} u {W..W+P}; every entry is then a 4-corner box sum
// (bcd_lag_assemble_kernel).  (2S-1)^2 lags x Hc x Wc products per plane instead of M^2/2 x H x W.
constexpr int kLagRB = 16;  // code rows per staged band

// Three lags (du, dv0..dv0+2) per thread: the products share the row-u value and a sliding window
// over row u+du, so a position costs two shared loads for three FMAs.
constexpr int kLagPerThread = 3;
template <int S>
__host__ __device__ constexpr int lag_threads() {
  return ((2 * S - 1) * ((2 * S - 1 + kLagPerThread - 1) / kLagPerThread) + 31) / 32 * 32;
}

template <int S>
__global__ void __launch_bounds__(lag_threads<S>(), 1)
bcd_lag_kernel(Geom g, const float* __restrict__ z, int nsplit, double* __restrict__ gq) {
  constexpr int P = S - 1;
  constexpr int NDV = 2 * S - 1;
  constexpr int NG = (NDV + kLagPerThread - 1) / kLagPerThread;
  constexpr int NL = NDV * NDV;
  constexpr int NCUT = 2 * S;
  constexpr int L = kLagPerThread;
  // rows [u0 - P, u0 + kLagRB + P) x columns [-P, Wc + P + L), fp64, zero outside the plane
  extern __shared__ double zb[];
  const int k = blockIdx.y, sp = blockIdx.x;
  const int t = threadIdx.x;
  const bool act = t < NDV * NG;
  const int du = act ? t / NG - P : 0;
  const int dv0 = act ? (t % NG) * L - P : 0;
  const int rows = kLagRB + 2 * P;
  const int pitch = g.Wc + 2 * P + L;
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  // column cuts: c_j = j (j <= P), W + j - S (j > P); row cuts likewise with H
  double Q[L][NCUT][NCUT];
#pragma unroll
  for (int l = 0; l < L; ++l)
#pragma unroll
    for (int i = 0; i < NCUT; ++i)
#pragma unroll
      for (int j = 0; j < NCUT; ++j) Q[l][i][j] = 0.0;
  const int n0 = static_cast<int>((static_cast<int64_t>(sp) * g.N) / nsplit);
  const int n1 = static_cast<int>((static_cast<int64_t>(sp + 1) * g.N) / nsplit);
  for (int n = n0; n < n1; ++n) {
    const float* zk = z + (static_cast<int64_t>(n) * g.K + k) * plane;
    double colacc[L][NCUT];  // sum over rows u < current of the row prefixes at the column cuts
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int j = 0; j < NCUT; ++j) colacc[l][j] = 0.0;
    int ri = 1;  // next row cut to capture (cut 0 is the empty prefix)
    for (int u0 = 0; u0 < g.Hc; u0 += kLagRB) {
      __syncthreads();
      for (int e = threadIdx.x; e < rows * pitch; e += blockDim.x) {
        const int rr = e / pitch, c = e - rr * pitch - P;
        const int u = u0 - P + rr;
        zb[e] = (u >= 0 && u < g.Hc && c >= 0 && c < g.Wc)
                    ? static_cast<double>(__ldg(zk + static_cast<int64_t>(u) * g.Wc + c)) : 0.0;
      }
      __syncthreads();
      if (!act) continue;
      const int ub = min(kLagRB, g.Hc - u0);
      for (int uu = 0; uu < ub; ++uu) {
        const double* r0 = zb + (uu + P) * pitch + P;             // row u, column 0
        const double* r1 = zb + (uu + P + du) * pitch + P + dv0;  // row u + du, column dv0 (zero padded)
        double rp[L];
#pragma unroll
        for (int l = 0; l < L; ++l) rp[l] = 0.0;
        double w0 = r1[0], w1 = r1[1], w2 = r1[2];
        int v = 0;
#pragma unroll
        for (int j = 1; j < NCUT; ++j) {
          const int cj = j <= P ? j : g.W + j - S;
          for (; v < cj; ++v) {
            const double x = r0[v];
            rp[0] = fma(x, w0, rp[0]);
            rp[1] = fma(x, w1, rp[1]);
            rp[2] = fma(x, w2, rp[2]);
            w0 = w1;
            w1 = w2;
            w2 = r1[v + 3];
          }
#pragma unroll
          for (int l = 0; l < L; ++l) colacc[l][j] += rp[l];
        }
        const int u = u0 + uu;
        // after row u: rows < u + 1 are in colacc; capture at the row cuts
        const int rcut = ri <= P ? ri : g.H + ri - S;
        if (ri < NCUT && u + 1 == rcut) {
#pragma unroll
          for (int l = 0; l < L; ++l)
#pragma unroll
            for (int j = 0; j < NCUT; ++j) Q[l][ri][j] += colacc[l][j];
          ++ri;
        }
      }
    }
  }
  if (act) {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int dv = dv0 + l;
      if (dv > P) continue;
      const int lag = (du + P) * NDV + (dv + P);
      double* out = gq + ((static_cast<int64_t>(k) * nsplit + sp) * NL + lag) * NCUT * NCUT;
#pragma unroll
      for (int i = 0; i < NCUT; ++i)
#pragma unroll
        for (int j = 0; j < NCUT; ++j) out[i * NCUT + j] = Q[l][i][j];
    }
  }
}

// C_kk entries from the prefix sums: E = Q(rh, ch) - Q(rl, ch) - Q(rh, cl) + Q(rl, cl) summed over the
// splits (fixed order), rl = P - a (cut a' = P - a), rh = P - a + H (cut S + P - a), cl / ch likewise
__global__ void bcd_lag_assemble_kernel(Geom g, const double* __restrict__ gq, int nsplit, double* __restrict__ cout) {
  const int S = g.S, P = g.P, M = S * S;
  const int NL = (2 * S - 1) * (2 * S - 1), NCUT = 2 * S;
  const int k = blockIdx.x;
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int t1 = e / M, t2 = e - t1 * M;
    const int a = t1 / S, b = t1 % S, a2 = t2 / S, b2 = t2 % S;
    const int lag = (a - a2 + P) * (2 * S - 1) + (b - b2 + P);
    const int rl = P - a, rh = S + P - a, cl = P - b, ch = S + P - b;
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const double* q = gq + ((static_cast<int64_t>(k) * nsplit + sp) * NL + lag) * NCUT * NCUT;
      s += (q[rh * NCUT + ch] - q[rl * NCUT + ch]) - (q[rh * NCUT + cl] - q[rl * NCUT + cl]);
    }
    cout[static_cast<int64_t>(k) * M * M + e] = s;
  }
}

// ================================================================ online surrogates (Eq.7 / Eq.8)
// SURVEY.md §8f NEXT-2; DESIGN.md §12.  C block-major [K][K][M][M], B [K][M].

// Lag-structured batch Gram of one filter pair (k1 <= k2, block q) folded straight into C (Eq.7):
// as bcd_lag_kernel with the products z_k1[u,v] z_k2[u+du, v+dv] of two planes, every thread (lag)
// then assembles the entries of its lag from the 4-corner box sums and writes
// C[k1][k2][t1][t2] = wo C + wn E (and the mirrored C[k2][k1][t2][t1]).
template <int S>
__global__ void __launch_bounds__(lag_threads<S>(), 1)
sur_lag_kernel(Geom g, const float* __restrict__ z, double wo, double wn, double* __restrict__ C) {
  constexpr int P = S - 1;
  constexpr int NDV = 2 * S - 1;
  constexpr int NG = (NDV + kLagPerThread - 1) / kLagPerThread;
  constexpr int NCUT = 2 * S;
  constexpr int M = S * S;
  constexpr int L = kLagPerThread;
  extern __shared__ double zb2[];  // [2][rows][pitch]: plane k1 rows u, plane k2 rows u+du (zero padded)
  const int q = blockIdx.x;
  int k1 = 0, rem = q;
  while (rem >= g.K - k1) {
    rem -= g.K - k1;
    ++k1;
  }
  const int k2 = k1 + rem;
  const int t = threadIdx.x;
  const bool act = t < NDV * NG;
  const int du = act ? t / NG - P : 0;
  const int dv0 = act ? (t % NG) * L - P : 0;
  const int rows = kLagRB + 2 * P;
  const int pitch = g.Wc + 2 * P + L;
  double* za = zb2;
  double* zc = zb2 + rows * pitch;
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  double Q[L][NCUT][NCUT];
#pragma unroll
  for (int l = 0; l < L; ++l)
#pragma unroll
    for (int i = 0; i < NCUT; ++i)
#pragma unroll
      for (int j = 0; j < NCUT; ++j) Q[l][i][j] = 0.0;
  for (int n = 0; n < g.N; ++n) {
    const float* z1 = z + (static_cast<int64_t>(n) * g.K + k1) * plane;
    const float* z2 = z + (static_cast<int64_t>(n) * g.K + k2) * plane;
    double colacc[L][NCUT];
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int j = 0; j < NCUT; ++j) colacc[l][j] = 0.0;
    int ri = 1;
    for (int u0 = 0; u0 < g.Hc; u0 += kLagRB) {
      __syncthreads();
      for (int e = threadIdx.x; e < rows * pitch; e += blockDim.x) {
        const int rr = e / pitch, c = e - rr * pitch - P;
        const int u = u0 - P + rr;
        const bool in = u >= 0 && u < g.Hc && c >= 0 && c < g.Wc;
        const int64_t off = static_cast<int64_t>(u) * g.Wc + c;
        za[e] = in ? static_cast<double>(__ldg(z1 + off)) : 0.0;
        zc[e] = in ? static_cast<double>(__ldg(z2 + off)) : 0.0;
      }
      __syncthreads();
      if (!act) continue;
      const int ub = min(kLagRB, g.Hc - u0);
      for (int uu = 0; uu < ub; ++uu) {
        const double* r0 = za + (uu + P) * pitch + P;
        const double* r1 = zc + (uu + P + du) * pitch + P + dv0;
        double rp[L];
#pragma unroll
        for (int l = 0; l < L; ++l) rp[l] = 0.0;
        double w0 = r1[0], w1 = r1[1], w2 = r1[2];
        int v = 0;
#pragma unroll
        for (int j = 1; j < NCUT; ++j) {
          const int cj = j <= P ? j : g.W + j - S;
          for (; v < cj; ++v) {
            const double x = r0[v];
            rp[0] = fma(x, w0, rp[0]);
            rp[1] = fma(x, w1, rp[1]);
            rp[2] = fma(x, w2, rp[2]);
            w0 = w1;
            w1 = w2;
            w2 = r1[v + 3];
          }
#pragma unroll
          for (int l = 0; l < L; ++l) colacc[l][j] += rp[l];
        }
        const int u = u0 + uu;
        const int rcut = ri <= P ? ri : g.H + ri - S;
        if (ri < NCUT && u + 1 == rcut) {
#pragma unroll
          for (int l = 0; l < L; ++l)
#pragma unroll
            for (int j = 0; j < NCUT; ++j) Q[l][ri][j] += colacc[l][j];
          ++ri;
        }
      }
    }
  }
  if (!act) return;
  // the entries of this thread's lags: (a, b) with a' = a - du, b' = b - dv inside [0, S)
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int dv = dv0 + l;
    if (dv > P) continue;
    for (int a = max(0, du); a < min(S, S + du); ++a)
      for (int b = max(0, dv); b < min(S, S + dv); ++b) {
        const int a2 = a - du, b2 = b - dv;
        const int rl = P - a, rh = S + P - a, cl = P - b, ch = S + P - b;
        const double E = (Q[l][rh][ch] - Q[l][rl][ch]) - (Q[l][rh][cl] - Q[l][rl][cl]);
        const int t1 = a * S + b, t2 = a2 * S + b2;
        double& c12 = C[((static_cast<int64_t>(k1) * g.K + k2) * M + t1) * M + t2];
        const double nv = wo * c12 + wn * E;
        c12 = nv;
        if (k1 != k2) C[((static_cast<int64_t>(k2) * g.K + k1) * M + t2) * M + t1] = nv;
      }
  }
}

// Batch Gram block (k1, k2), k1 <= k2 (pair index q in the upper triangle, row by row): partial over
// the images of split sp, all M x M entries, 4x4 tiles, processed in passes of 2 tiles per thread.
__global__ void __launch_bounds__(kGramThreads) sur_gram_kernel(Geom g, const float* __restrict__ z, int nsplit,
                                                                double* __restrict__ pp) {
  extern __shared__ double zz[];  // [2][kGramBR + P][Wc] + 1 zero
  const int q = blockIdx.y, sp = blockIdx.x;
  int k1 = 0, rem = q;
  while (rem >= g.K - k1) {
    rem -= g.K - k1;
    ++k1;
  }
  const int k2 = k1 + rem;
  const int M = g.S * g.S;
  const int NT = (M + 3) / 4;
  const int rows = kGramBR + g.P;
  const int half = rows * g.Wc;
  const int zero_at = 2 * half;
  double* z1s = zz;
  double* z2s = zz + half;
  const int n0 = static_cast<int>((static_cast<int64_t>(sp) * g.N) / nsplit);
  const int n1 = static_cast<int>((static_cast<int64_t>(sp + 1) * g.N) / nsplit);
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc;
  double* out = pp + (static_cast<int64_t>(q) * nsplit + sp) * M * M;
  if (threadIdx.x == 0) zz[zero_at] = 0.0;
  for (int pass = 0; pass * 2 * kGramThreads < NT * NT; ++pass) {
    int off1[2][4], off2[2][4], T1v[2], T2v[2];
    bool own[2];
    for (int h = 0; h < 2; ++h) {
      const int id = pass * 2 * kGramThreads + h * kGramThreads + threadIdx.x;
      own[h] = id < NT * NT;
      T1v[h] = own[h] ? id / NT : 0;
      T2v[h] = own[h] ? id % NT : 0;
      for (int e = 0; e < 4; ++e) {
        const int t1 = 4 * T1v[h] + e, t2 = 4 * T2v[h] + e;
        off1[h][e] = t1 < M ? (g.P - t1 / g.S) * g.Wc + (g.P - t1 % g.S) : -1;
        off2[h][e] = t2 < M ? half + (g.P - t2 / g.S) * g.Wc + (g.P - t2 % g.S) : -1;
      }
    }
    double acc[2][4][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[h][a][b] = 0.0;
    for (int n = n0; n < n1; ++n) {
      const float* za = z + (static_cast<int64_t>(n) * g.K + k1) * plane;
      const float* zb = z + (static_cast<int64_t>(n) * g.K + k2) * plane;
      for (int i0 = 0; i0 < g.H; i0 += kGramBR) {
        __syncthreads();
        const int nr = min(rows, g.Hc - i0);
        for (int e = threadIdx.x; e < half; e += kGramThreads) {
          const int rr = e / g.Wc;
          const bool in = rr < nr;
          z1s[e] = in ? static_cast<double>(__ldg(za + static_cast<int64_t>(i0) * g.Wc + e)) : 0.0;
          z2s[e] = in ? static_cast<double>(__ldg(zb + static_cast<int64_t>(i0) * g.Wc + e)) : 0.0;
        }
        __syncthreads();
        const int ib = min(kGramBR, g.H - i0);
        for (int ii = 0; ii < ib; ++ii)
          for (int j = 0; j < g.W; ++j) {
            const int base = ii * g.Wc + j;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (!own[h]) continue;
              double x1[4], x2[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                x1[e] = zz[off1[h][e] >= 0 ? base + off1[h][e] : zero_at];
                x2[e] = zz[off2[h][e] >= 0 ? base + off2[h][e] : zero_at];
              }
#pragma unroll
              for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[h][a][b] = fma(x1[a], x2[b], acc[h][a][b]);
            }
          }
      }
    }
    for (int h = 0; h < 2; ++h) {
      if (!own[h]) continue;
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
          const int t1 = 4 * T1v[h] + a, t2 = 4 * T2v[h] + b;
          if (t1 < M && t2 < M) out[static_cast<int64_t>(t1) * M + t2] = acc[h][a][b];
        }
    }
  }
}

// C[k1][k2] = wo C + wn sum_sp pp, mirrored into C[k2][k1] (fixed order over the splits)
__global__ void sur_fold_kernel(Geom g, const double* __restrict__ pp, int nsplit, double wo, double wn,
                                double* __restrict__ C) {
  const int M = g.S * g.S;
  const int64_t npairs = static_cast<int64_t>(g.K) * (g.K + 1) / 2;
  const int64_t total = npairs * M * M;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / (M * M);
    const int rem2 = static_cast<int>(e - q * M * M);
    const int t1 = rem2 / M, t2 = rem2 - t1 * M;
    int k1 = 0;
    int64_t rem = q;
    while (rem >= g.K - k1) {
      rem -= g.K - k1;
      ++k1;
    }
    const int k2 = k1 + static_cast<int>(rem);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += pp[(q * nsplit + sp) * M * M + rem2];
    double& c = C[((static_cast<int64_t>(k1) * g.K + k2) * M + t1) * M + t2];
    c = wo * c + wn * s;
    if (k1 != k2) C[((static_cast<int64_t>(k2) * g.K + k1) * M + t2) * M + t1] = c;
  }
}

// B[k] = wo B[k] + wn gk (gk = sum_n Z_nk^T x_n from bcd_gk_kernel with r := x)
__global__ void sur_bfold_kernel(int M, int k, const double* __restrict__ gk, double wo, double wn,
                                 double* __restrict__ B) {
  const int t = threadIdx.x;
  if (t < M) B[static_cast<int64_t>(k) * M + t] = wo * B[static_cast<int64_t>(k) * M + t] + wn * gk[t];
}

// diag[k] = C[k][k] (contiguous [K][M][M] for bcd_inverse_kernel)
__global__ void sur_diag_kernel(Geom g, const double* __restrict__ C, double* __restrict__ diag) {
  const int M = g.S * g.S;
  const int k = blockIdx.x;
  for (int e = threadIdx.x; e < M * M; e += blockDim.x)
    diag[static_cast<int64_t>(k) * M * M + e] = C[(static_cast<int64_t>(k) * g.K + k) * M * M + e];
}

// g[t] = sum_k2 sum_t2 C[k][k2][t][t2] d[k2][t2] - B[k][t]: block t (fixed-order tree reduction)
__global__ void sur_grad_kernel(Geom g, int k, const double* __restrict__ C, const double* __restrict__ B,
                                const float* __restrict__ d, double* __restrict__ gk) {
  __shared__ double red[32];
  const int M = g.S * g.S;
  const int t = blockIdx.x;
  const int64_t KM = static_cast<int64_t>(g.K) * M;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < KM; e += blockDim.x) {
    const int64_t k2 = e / M;
    const int t2 = static_cast<int>(e - k2 * M);
    s = fma(C[((static_cast<int64_t>(k) * g.K + k2) * M + t) * M + t2], static_cast<double>(d[e]), s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullB, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
    gk[t] = tot - B[static_cast<int64_t>(k) * M + t];
  }
}

}  // namespace

int bcd_gram_splits(const Geom& g) {
  int ns = (148 * 2 + g.K - 1) / g.K;  // independent of the local image count (same on every rank)
  if (ns < 1) ns = 1;
  return ns;
}
int bcd_gk_blocks(const Geom& g) { return g.N * ((g.H + kGkBR - 1) / kGkBR); }

cudaError_t launch_bcd_gram(const Geom& g, const float* z, double* gpart, cudaStream_t st) {
  const int ns = bcd_gram_splits(g);
  const size_t smem = sizeof(double) * ((kGramBR + g.P) * g.Wc + 1);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bcd_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  bcd_gram_kernel<<<dim3(ns, g.K), kGramThreads, smem, st>>>(g, z, ns, gpart);
  return cudaGetLastError();
}

cudaError_t launch_bcd_inverse(const Geom& g, const double* gpart, double ridge_rel, double* ainv, uint8_t* flags,
                               cudaStream_t st) {
  const int M = g.S * g.S;
  const size_t smem2 = sizeof(double) * M * M;
  if (smem2 > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bcd_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem2));
    if (e != cudaSuccess) return e;
  }
  bcd_inverse_kernel<<<g.K, 128, smem2, st>>>(g, gpart, bcd_gram_splits(g), ridge_rel, ainv, flags);
  return cudaGetLastError();
}

cudaError_t launch_bcd_gk(const Geom& g, int k, const float* z, const float* r, double* part, double* gk,
                          cudaStream_t st) {
  const int M = g.S * g.S;
  const int nb = bcd_gk_blocks(g);
  if (nb > 0) {
    const size_t smem = sizeof(double) * ((kGkBR + g.P) * g.Wc + kGkBR * g.W);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(bcd_gk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    bcd_gk_kernel<<<nb, 128, smem, st>>>(g, k, z, r, part);
  }
  bcd_gsum_kernel<<<(M + 7) / 8, 256, 0, st>>>(M, part, nb, gk);
  return cudaGetLastError();
}

cudaError_t launch_bcd_update(const Geom& g, int k, const double* gk, const double* ainv, const uint8_t* flags,
                              float* d, double* dl, const float* z, float* r, cudaStream_t st) {
  bcd_update_kernel<<<1, 128, 0, st>>>(g, k, gk, ainv, flags, d, dl);
  const int64_t npx = static_cast<int64_t>(g.N) * g.H * g.W;
  if (npx > 0) {
    int64_t rb = (npx + 255) / 256;
    if (rb > 148 * 8) rb = 148 * 8;
    bcd_resid_kernel<<<static_cast<unsigned>(rb), 256, 0, st>>>(g, k, z, dl, r);
  }
  return cudaGetLastError();
}

bool bcd_lag_supported(const Geom& g) { return g.H > g.P && g.W > g.P && g.S >= 1 && g.S <= 11 && (g.S & 1); }

cudaError_t launch_bcd_lag_gram(const Geom& g, const float* z, double* gq, double* cfull, cudaStream_t st) {
  const int ns = bcd_gram_splits(g);
  const size_t smem = sizeof(double) * (kLagRB + 2 * g.P) * (g.Wc + 2 * g.P + kLagPerThread);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto sz) -> cudaError_t {
    constexpr int SS = decltype(sz)::value;
    constexpr int NT = lag_threads<SS>();
    if (smem > 48 * 1024) {
      cudaError_t er = cudaFuncSetAttribute(bcd_lag_kernel<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem));
      if (er != cudaSuccess) return er;
    }
    if (g.N > 0) bcd_lag_kernel<SS><<<dim3(ns, g.K), NT, smem, st>>>(g, z, ns, gq);
    else cudaMemsetAsync(gq, 0, sizeof(double) * g.K * ns * (2 * SS - 1) * (2 * SS - 1) * 4 * SS * SS, st);
    return cudaGetLastError();
  };
  switch (g.S) {
    case 1: e = go(std::integral_constant<int, 1>{}); break;
    case 3: e = go(std::integral_constant<int, 3>{}); break;
    case 5: e = go(std::integral_constant<int, 5>{}); break;
    case 7: e = go(std::integral_constant<int, 7>{}); break;
    case 9: e = go(std::integral_constant<int, 9>{}); break;
    case 11: e = go(std::integral_constant<int, 11>{}); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  bcd_lag_assemble_kernel<<<g.K, 256, 0, st>>>(g, gq, ns, cfull);
  return cudaGetLastError();
}

size_t bcd_lag_bytes(const Geom& g) {
  const int ns = bcd_gram_splits(g);
  return sizeof(double) * static_cast<size_t>(g.K) * ns * (2 * g.S - 1) * (2 * g.S - 1) * 4 * g.S * g.S;
}

cudaError_t launch_bcd_inverse_full(const Geom& g, const double* cfull, double ridge_rel, double* ainv,
                                    uint8_t* flags, cudaStream_t st) {
  const int M = g.S * g.S;
  const size_t smem2 = sizeof(double) * M * M;
  if (smem2 > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bcd_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem2));
    if (e != cudaSuccess) return e;
  }
  bcd_inverse_kernel<<<g.K, 128, smem2, st>>>(g, cfull, 1, ridge_rel, ainv, flags);
  return cudaGetLastError();
}

int sur_gram_splits(const Geom& g) {
  const int64_t np = static_cast<int64_t>(g.K) * (g.K + 1) / 2;
  int ns = static_cast<int>((148 * 2 + np - 1) / np);
  if (ns < 1) ns = 1;
  return ns;
}

cudaError_t launch_sur_update(const Geom& g, const float* x, const float* z, double* pp, double* part, double* gk,
                              double wo, double wn, double* C, double* B, cudaStream_t st) {
  const int ns = sur_gram_splits(g);
  const int64_t np = static_cast<int64_t>(g.K) * (g.K + 1) / 2;
  const int M = g.S * g.S;
  if (pp == nullptr) {
    // lag-structured path (bcd_lag_supported): one block per filter pair, folded in place
    const size_t smem = sizeof(double) * 2 * (kLagRB + 2 * g.P) * (g.Wc + 2 * g.P + kLagPerThread);
    auto go = [&](auto sz) -> cudaError_t {
      constexpr int SS = decltype(sz)::value;
      constexpr int NT = lag_threads<SS>();
      if (smem > 48 * 1024) {
        cudaError_t er = cudaFuncSetAttribute(sur_lag_kernel<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem));
        if (er != cudaSuccess) return er;
      }
      sur_lag_kernel<SS><<<static_cast<unsigned>(np), NT, smem, st>>>(g, z, wo, wn, C);
      return cudaGetLastError();
    };
    cudaError_t e = cudaSuccess;
    switch (g.S) {
      case 1: e = go(std::integral_constant<int, 1>{}); break;
      case 3: e = go(std::integral_constant<int, 3>{}); break;
      case 5: e = go(std::integral_constant<int, 5>{}); break;
      case 7: e = go(std::integral_constant<int, 7>{}); break;
      case 9: e = go(std::integral_constant<int, 9>{}); break;
      case 11: e = go(std::integral_constant<int, 11>{}); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    for (int k = 0; k < g.K; ++k) {
      e = launch_bcd_gk(g, k, z, x, part, gk, st);
      if (e != cudaSuccess) return e;
      sur_bfold_kernel<<<1, 128, 0, st>>>(M, k, gk, wo, wn, B);
    }
    return cudaGetLastError();
  }
  if (g.N > 0) {
    const size_t smem = sizeof(double) * (2 * (kGramBR + g.P) * g.Wc + 1);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(sur_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    sur_gram_kernel<<<dim3(ns, static_cast<unsigned>(np)), kGramThreads, smem, st>>>(g, z, ns, pp);
  } else {
    cudaMemsetAsync(pp, 0, sizeof(double) * np * ns * M * M, st);
  }
  int64_t fb = (np * M * M + 255) / 256;
  if (fb > 148 * 16) fb = 148 * 16;
  sur_fold_kernel<<<static_cast<unsigned>(fb), 256, 0, st>>>(g, pp, ns, wo, wn, C);
  for (int k = 0; k < g.K; ++k) {
    cudaError_t e = launch_bcd_gk(g, k, z, x, part, gk, st);
    if (e != cudaSuccess) return e;
    sur_bfold_kernel<<<1, 128, 0, st>>>(M, k, gk, wo, wn, B);
  }
  return cudaGetLastError();
}

cudaError_t launch_sur_prepare(const Geom& g, const double* C, double* diag, double ridge_rel, double* ainv,
                               uint8_t* flags, cudaStream_t st) {
  sur_diag_kernel<<<g.K, 256, 0, st>>>(g, C, diag);
  const int M = g.S * g.S;
  const size_t smem2 = sizeof(double) * M * M;
  if (smem2 > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bcd_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem2));
    if (e != cudaSuccess) return e;
  }
  bcd_inverse_kernel<<<g.K, 128, smem2, st>>>(g, diag, 1, ridge_rel, ainv, flags);
  return cudaGetLastError();
}

cudaError_t launch_sur_filter(const Geom& g, int k, const double* C, const double* B, const double* ainv,
                              const uint8_t* flags, float* d, double* gk, double* dl, cudaStream_t st) {
  const int M = g.S * g.S;
  sur_grad_kernel<<<M, 256, 0, st>>>(g, k, C, B, d, gk);
  bcd_update_kernel<<<1, 128, 0, st>>>(g, k, gk, ainv, flags, d, dl);
  return cudaGetLastError();
}

}  // namespace csc

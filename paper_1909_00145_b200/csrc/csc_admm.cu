// csc_admm.cu -- kernels of the ADMM masked-LASSO code solver (PAPER.md
// P:303-321 §3.2): the paper's own code update, as an alternative to the one-step prox-gradient
// code step of the hot path (reading R1).
//
// Per image n the selected codes w (mask M^t, Eq.2) solve Eq.3 by scaled ADMM (A1-A6):
//   b = x - D z_fix,  A = D M^T,  w = y = z[M], u = 0, then 10 times
//   CG (n_cg steps, warm start w) on (A^T A + rho I) w = A^T b + rho (y - u)
//   w^ = alpha w + (1 - alpha) y,   y = S_{lam/rho}(w^ + u),   u = u + w^ - y
// and z[M] = y.  The vectors live in code-shaped buffers (0 off the mask); A v is the dense pass
// of csc_api.cu (tensor cores) and A^T e is masked_dtr_kernel below.  CG scalars are per image,
// reduced in fp64 in a fixed order (deterministic), and never leave the device.
#include "csc_internal.cuh"

#include <cstdint>
#include <cuda_runtime.h>

namespace csc {
namespace {

constexpr unsigned kFullA = 0xffffffffu;
constexpr int kAdmmThreads = 256;

__device__ __forceinline__ bool mbit(const uint32_t* __restrict__ bits, int64_t l) {
  return (__ldg(bits + (l >> 5)) >> (l & 31)) & 1u;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullA, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// blocks: grid (nb, N); block (b, n) covers codes l = b*blockDim + tid, stride nb*blockDim, of image n.

// out = M (D^T e) + rho * v   (v may be null: rho term dropped);  part[n][b] = sum v * out (if dot)
__global__ void masked_dtr_kernel(Geom g, const float* __restrict__ e, const float* __restrict__ d,
                                  const uint32_t* __restrict__ bits, const float* __restrict__ v, float rho,
                                  float sign, float* __restrict__ out, double* __restrict__ part) {
  const int n = blockIdx.y;
  const int64_t plane = static_cast<int64_t>(g.Hc) * g.Wc, nc = plane * g.K;
  const float* en = e + static_cast<int64_t>(n) * g.H * g.W;
  double acc = 0.0;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    float o = 0.f;
    if (mbit(bits, l)) {
      const int k = static_cast<int>(l / plane);
      const int64_t pp = l - static_cast<int64_t>(k) * plane;
      const int u = static_cast<int>(pp / g.Wc), vv = static_cast<int>(pp - static_cast<int64_t>(u) * g.Wc);
      const float* dk = d + static_cast<int64_t>(k) * g.S * g.S;
      float c = 0.f;
      for (int a = 0; a < g.S; ++a) {
        const int i = u - g.P + a;
        if (i < 0 || i >= g.H) continue;
        for (int b = 0; b < g.S; ++b) {
          const int j = vv - g.P + b;
          if (j < 0 || j >= g.W) continue;
          c = fmaf(__ldg(dk + a * g.S + b), __ldg(en + static_cast<int64_t>(i) * g.W + j), c);
        }
      }
      o = sign * c;
      if (v != nullptr) o = fmaf(rho, v[gi], o);
      if (part != nullptr && v != nullptr) acc += static_cast<double>(v[gi]) * static_cast<double>(o);
    }
    out[gi] = o;
  }
  if (part != nullptr) {
    const double t = block_sum(acc);
    if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
  }
}

// W = Y = z on M (0 off M), U = 0, Zf = z off M (0 on M)
__global__ void admm_init_kernel(Geom g, const float* __restrict__ z, const uint32_t* __restrict__ bits,
                                 float* __restrict__ W, float* __restrict__ Y, float* __restrict__ U,
                                 float* __restrict__ Zf) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    const bool m = mbit(bits, l);
    const float zv = z[gi];
    W[gi] = m ? zv : 0.f;
    Y[gi] = m ? zv : 0.f;
    U[gi] = 0.f;
    Zf[gi] = m ? 0.f : zv;
  }
}

// CG start: R = ATB + rho (Y - U) - Q ,  PV = R,  part[n][b] = sum R^2   (all zero off M)
__global__ void cg_start_kernel(Geom g, const float* __restrict__ ATB, const float* __restrict__ Y,
                                const float* __restrict__ U, const float* __restrict__ Q, float rho,
                                float* __restrict__ R, float* __restrict__ PV, double* __restrict__ part) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  double acc = 0.0;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    const float r = ATB[gi] + rho * (Y[gi] - U[gi]) - Q[gi];  // zero off M: every term is
    R[gi] = r;
    PV[gi] = r;
    acc += static_cast<double>(r) * static_cast<double>(r);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

// per image: s[n] = sum_b part[n][b] (fixed order)
__global__ void image_sum_kernel(const double* __restrict__ part, int nb, int N, double* __restrict__ out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[static_cast<int64_t>(n) * nb + b];
  out[n] = s;
}

// CG step: a = rr / pq (0 if rr == 0 or pq <= 0), W += a PV, R -= a Q, part = sum R^2
__global__ void cg_step_kernel(Geom g, const double* __restrict__ rr, const double* __restrict__ pq,
                               float* __restrict__ W, float* __restrict__ R, const float* __restrict__ PV,
                               const float* __restrict__ Q, double* __restrict__ part) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  const double r0 = rr[n], d0 = pq[n];
  const float a = (r0 > 0.0 && d0 > 0.0) ? static_cast<float>(r0 / d0) : 0.f;
  double acc = 0.0;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    W[gi] = fmaf(a, PV[gi], W[gi]);
    const float r = fmaf(-a, Q[gi], R[gi]);
    R[gi] = r;
    acc += static_cast<double>(r) * static_cast<double>(r);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[static_cast<int64_t>(n) * gridDim.x + blockIdx.x] = t;
}

// CG direction: beta = rr_new / rr (0 if rr == 0), PV = R + beta PV; rr <- rr_new
__global__ void cg_dir_kernel(Geom g, double* __restrict__ rr, const double* __restrict__ rr_new,
                              const float* __restrict__ R, float* __restrict__ PV) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  const double r0 = rr[n], r1 = rr_new[n];
  const float beta = r0 > 0.0 ? static_cast<float>(r1 / r0) : 0.f;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    PV[gi] = fmaf(beta, PV[gi], R[gi]);
  }
}

__global__ void rr_copy_kernel(double* __restrict__ rr, const double* __restrict__ rr_new, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < N) rr[n] = rr_new[n];
}

// w^ = alpha W + (1 - alpha) Y;  Y' = S(w^ + U, kappa) (+0.0 in the dead zone);  U += w^ - Y';  Y = Y'
__global__ void admm_update_kernel(Geom g, const uint32_t* __restrict__ bits, const float* __restrict__ W,
                                   float* __restrict__ Y, float* __restrict__ U, float alpha, float kappa) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!mbit(bits, l)) continue;
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    const float wh = fmaf(alpha, W[gi], (1.f - alpha) * Y[gi]);
    const float q = wh + U[gi];
    const float yn = q > kappa ? q - kappa : (q < -kappa ? q + kappa : 0.f);
    U[gi] = U[gi] + (wh - yn);
    Y[gi] = yn;
  }
}

// z[M] = Y, z unchanged off M; the max|z| bound of the fp16 dense pass is raised with the new codes
__global__ void admm_finish_kernel(Geom g, const uint32_t* __restrict__ bits, const float* __restrict__ Y,
                                   float* __restrict__ z, uint32_t* __restrict__ zmax) {
  const int n = blockIdx.y;
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  uint32_t m = 0u;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!mbit(bits, l)) continue;
    const int64_t gi = static_cast<int64_t>(n) * nc + l;
    z[gi] = Y[gi];
    m = max(m, __float_as_uint(fabsf(Y[gi])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFullA, m, o));
  if ((threadIdx.x & 31) == 0 && zmax != nullptr && m != 0u) atomicMax(zmax, m);
}

}  // namespace

int admm_blocks_per_image(const Geom& g) {
  const int64_t nc = static_cast<int64_t>(g.Hc) * g.Wc * g.K;
  int64_t nb = (nc + kAdmmThreads * 8 - 1) / (kAdmmThreads * 8);
  int64_t cap = (148 * 8 + (g.N > 0 ? g.N : 1) - 1) / (g.N > 0 ? g.N : 1);
  if (nb > cap) nb = cap;
  if (nb < 1) nb = 1;
  return static_cast<int>(nb);
}

cudaError_t launch_masked_dtr(const Geom& g, const float* e, const float* d, const uint32_t* bits, const float* v,
                              float rho, float sign, float* out, double* part, cudaStream_t st) {
  const dim3 grid(admm_blocks_per_image(g), g.N);
  masked_dtr_kernel<<<grid, kAdmmThreads, 0, st>>>(g, e, d, bits, v, rho, sign, out, part);
  return cudaGetLastError();
}
cudaError_t launch_admm_init(const Geom& g, const float* z, const uint32_t* bits, float* W, float* Y, float* U,
                             float* Zf, cudaStream_t st) {
  admm_init_kernel<<<dim3(admm_blocks_per_image(g), g.N), kAdmmThreads, 0, st>>>(g, z, bits, W, Y, U, Zf);
  return cudaGetLastError();
}
cudaError_t launch_cg_start(const Geom& g, const float* ATB, const float* Y, const float* U, const float* Q,
                            float rho, float* R, float* PV, double* part, double* rr, cudaStream_t st) {
  const int nb = admm_blocks_per_image(g);
  cg_start_kernel<<<dim3(nb, g.N), kAdmmThreads, 0, st>>>(g, ATB, Y, U, Q, rho, R, PV, part);
  image_sum_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(part, nb, g.N, rr);
  return cudaGetLastError();
}
cudaError_t launch_image_sum(const Geom& g, const double* part, double* out, cudaStream_t st) {
  image_sum_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(part, admm_blocks_per_image(g), g.N, out);
  return cudaGetLastError();
}
cudaError_t launch_cg_step(const Geom& g, const double* rr, const double* pq, float* W, float* R, const float* PV,
                           const float* Q, double* part, double* rr_new, cudaStream_t st) {
  const int nb = admm_blocks_per_image(g);
  cg_step_kernel<<<dim3(nb, g.N), kAdmmThreads, 0, st>>>(g, rr, pq, W, R, PV, Q, part);
  image_sum_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(part, nb, g.N, rr_new);
  return cudaGetLastError();
}
cudaError_t launch_cg_dir(const Geom& g, double* rr, const double* rr_new, const float* R, float* PV,
                          cudaStream_t st) {
  cg_dir_kernel<<<dim3(admm_blocks_per_image(g), g.N), kAdmmThreads, 0, st>>>(g, rr, rr_new, R, PV);
  rr_copy_kernel<<<(g.N + 127) / 128, 128, 0, st>>>(rr, rr_new, g.N);
  return cudaGetLastError();
}
cudaError_t launch_admm_update(const Geom& g, const uint32_t* bits, const float* W, float* Y, float* U, float alpha,
                               float kappa, cudaStream_t st) {
  admm_update_kernel<<<dim3(admm_blocks_per_image(g), g.N), kAdmmThreads, 0, st>>>(g, bits, W, Y, U, alpha, kappa);
  return cudaGetLastError();
}
cudaError_t launch_admm_finish(const Geom& g, const uint32_t* bits, const float* Y, float* z, uint32_t* zmax,
                               cudaStream_t st) {
  admm_finish_kernel<<<dim3(admm_blocks_per_image(g), g.N), kAdmmThreads, 0, st>>>(g, bits, Y, z, zmax);
  return cudaGetLastError();
}

}  // namespace csc

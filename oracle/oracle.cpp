// oracle/oracle.cpp -- CPU ORACLE FOR THE STOCHASTIC SPATIAL-DOMAIN CSC HOT PATH.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  The
// product path (paper_1909_00145_b200/) never links, imports or executes it,
// and this file shares no code, header, table or constant generator with it.
//
// Plain nested loops in the paper's order and notation.  State (x, d, z, r) is
// stored in T (float for parity with the GPU, double for the exact-arithmetic
// pins); every sum accumulates in double; each stored value is rounded once.
//
// Citations: P:n = PAPER.md line n (arxiv 1909.00145 LaTeX), with section /
// equation.  Readings R1..R9 and #1..#17 are listed in DESIGN.md §3.
//
// Notation (§2-3): N images x_n (H x W), K filters d_k (s x s,
// M = s^2), codes z_{n,k} of (H+s-1) x (W+s-1) (reading R3: "valid" true
// convolution, non-circular boundary), P = s-1.
//
// Pinned by tests/test_oracle_*.py (curand Philox, dense Toeplitz brute force,
// scipy convolve2d/correlate2d, adjoint identities, closed-form shrinkage,
// textbook ISTA at p=1, monotone descent, 1-D line-search optimality, numpy FFT
// for the DTFT bound).  The 50-iteration trajectory as a whole is "parity
// unpinned" beyond those pins: the paper prints no per-iteration value.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <omp.h>

namespace {

struct Dims {
  int64_t N, K, s, H, W, Hc, Wc, P;
  Dims(int64_t N_, int64_t K_, int64_t s_, int64_t H_, int64_t W_)
      : N(N_), K(K_), s(s_), H(H_), W(W_), Hc(H_ + s_ - 1), Wc(W_ + s_ - 1), P(s_ - 1) {}
  int64_t xi(int64_t n, int64_t i, int64_t j) const { return (n * H + i) * W + j; }
  int64_t di(int64_t k, int64_t a, int64_t b) const { return (k * s + a) * s + b; }
  int64_t zi(int64_t n, int64_t k, int64_t u, int64_t v) const {
    return ((n * K + k) * Hc + u) * Wc + v;
  }
};

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written from the
// algorithm: 10 rounds of  (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
// c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0), with the Weyl key bump (W0, W1)
// between rounds.  Pinned bit-exact against curand_Philox4x32_10.
// ---------------------------------------------------------------------------
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += W0; k1 += W1; }
    const uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    const uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Domain tag of the mask counter (reading R4 / DESIGN.md #13): the 4th counter
// word.  Arbitrary, chosen once ("CSCM").
const uint32_t kMaskTag = 0x4353434Du;

// thr = floor(p * 2^32) in double, as uint64 (p = 1 -> 2^32: everything selected,
// M^t = identity).
uint64_t mask_threshold(double p) { return (uint64_t)std::floor(p * 4294967296.0); }

// Eq.2, reading R4/R5: i.i.d. Bernoulli(p) per code coordinate
// l = (k*Hc + u)*Wc + v, one mask per iteration t shared by all images.
bool mask_bit(uint64_t seed, uint32_t t, uint64_t l, uint64_t thr) {
  const uint64_t q = l >> 2;
  const uint32_t ctr[4] = {(uint32_t)(q & 0xffffffffu), (uint32_t)(q >> 32), t, kMaskTag};
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t w[4];
  philox4x32_10(ctr, key, w);
  return (uint64_t)w[l & 3] < thr;
}

// Block-structured variant (a labelled deviation from the per-entry
// Bernoulli sampling of Eq.2; reading E5): one Bernoulli(p) draw per aligned
// block of 8 consecutive coordinates b = l >> 3 (one 32-B sector of fp32 codes), word b & 3 of
// Philox(ctr = {q lo, q hi, t, kSectorTag}, q = b >> 2).
const uint32_t kSectorTag = 0x43534253u;  // "CSBS"
bool mask_bit_sector8(uint64_t seed, uint32_t t, uint64_t l, uint64_t thr) {
  const uint64_t b = l >> 3, q = b >> 2;
  const uint32_t ctr[4] = {(uint32_t)(q & 0xffffffffu), (uint32_t)(q >> 32), t, kSectorTag};
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t w[4];
  philox4x32_10(ctr, key, w);
  return (uint64_t)w[b & 3] < thr;
}
inline bool mask_bit_mode(int mode, uint64_t seed, uint32_t t, uint64_t l, uint64_t thr) {
  return mode == 1 ? mask_bit_sector8(seed, t, l, thr) : mask_bit(seed, t, l, thr);
}

// Dz - x  (Sec.3.1 P:191-197 "D z = sum_k d_k * z_k", fit term of Eq.1):
//   r[n,i,j] = sum_k sum_{a,b} d[k,a,b] z[n,k,i+P-a,j+P-b] - x[n,i,j]
// a "valid" true convolution: every tap lands inside the code map.
template <typename T>
void residual(const Dims& D, const T* x, const T* d, const T* z, T* r) {
  // every output pixel is an independent fp64 sum: rows (n, i) are spread over the threads
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t i = 0; i < D.H; ++i)
      for (int64_t j = 0; j < D.W; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < D.K; ++k)
          for (int64_t a = 0; a < D.s; ++a)
            for (int64_t b = 0; b < D.s; ++b)
              acc += (double)d[D.di(k, a, b)] * (double)z[D.zi(n, k, i + D.P - a, j + D.P - b)];
        r[D.xi(n, i, j)] = (T)(acc - (x ? (double)x[D.xi(n, i, j)] : 0.0));
      }
}

// (D^T r)[n,k,u,v] = sum_{a,b} d[k,a,b] r[n, u-P+a, v-P+b]  (r == 0 outside the
// image): the gradient of the fit term of Eq.3 w.r.t. code (k,u,v).
inline double dtr_at(const Dims& D, const double* dk, const double* rn, int64_t u, int64_t v) {
  double c = 0.0;
  for (int64_t a = 0; a < D.s; ++a) {
    const int64_t i = u - D.P + a;
    if (i < 0 || i >= D.H) continue;
    for (int64_t b = 0; b < D.s; ++b) {
      const int64_t j = v - D.P + b;
      if (j < 0 || j >= D.W) continue;
      c += dk[a * D.s + b] * rn[i * D.W + j];
    }
  }
  return c;
}

// D^T r for every code coordinate (all n, k, u, v), stored in T.
template <typename T>
void dtr_all(const Dims& D, const T* d, const T* r, T* out) {
  std::vector<double> dd((size_t)(D.K * D.s * D.s)), rd((size_t)(D.N * D.H * D.W));
  for (size_t q = 0; q < dd.size(); ++q) dd[q] = (double)d[q];
  for (size_t q = 0; q < rd.size(); ++q) rd[q] = (double)r[q];
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t k = 0; k < D.K; ++k)
      for (int64_t u = 0; u < D.Hc; ++u)
        for (int64_t v = 0; v < D.Wc; ++v)
          out[D.zi(n, k, u, v)] = (T)dtr_at(D, &dd[k * D.s * D.s], &rd[n * D.H * D.W], u, v);
}

// Soft threshold, the prox of kappa*||.||_1 ("point-wise shrinkage"):
// S(w,kappa) = w-kappa (w>kappa), w+kappa (w<-kappa), +0.0 otherwise (#12).
inline double soft_threshold(double w, double kappa) {
  if (w > kappa) return w - kappa;
  if (w < -kappa) return w + kappa;
  return 0.0;
}

// Lipschitz bound of the code gradient (reading R8, #7):
//   L_D = max_{m1,m2 in [0,64)} sum_k | sum_{a,b} d[k,a,b] e^{-2 pi i (a m1 + b m2)/64} |^2
template <typename T>
double lipschitz_dtft(const Dims& D, const T* d) {
  const int G = 64;
  // e^{-2 pi i n/64}, n = 0..63: the same cos/sin values the direct formula evaluates,
  // tabulated once (the exponent (a m1 + b m2) is taken mod 64).
  double cs[G], sn[G];
  for (int q = 0; q < G; ++q) {
    const double ang = -2.0 * M_PI * (double)q / (double)G;
    cs[q] = std::cos(ang);
    sn[q] = std::sin(ang);
  }
  double best = 0.0;
  for (int m1 = 0; m1 < G; ++m1)
    for (int m2 = 0; m2 < G; ++m2) {
      double tot = 0.0;
      for (int64_t k = 0; k < D.K; ++k) {
        double re = 0.0, im = 0.0;
        for (int64_t a = 0; a < D.s; ++a)
          for (int64_t b = 0; b < D.s; ++b) {
            const int q = (int)((a * m1 + b * m2) % G);
            const double v = (double)d[D.di(k, a, b)];
            re += v * cs[q];
            im += v * sn[q];
          }
        tot += re * re + im * im;
      }
      best = std::max(best, tot);
    }
  return best;
}

// One masked proximal-gradient step on the codes (reading R1): Eq.3
// restricted by M^t (Eq.2) and upsampled in place (Eq.4, reading R2: unsampled
// codes keep their values).
//
// Step rule (step_z == 0): eso == 0: tau = 1/L_D for every code (reading R8).  eso != 0: the
// expected-separable-overapproximation step of parallel coordinate descent under independent
// Bernoulli(p) sampling (P:620-623 cites the mini-batch coordinate
// descent literature; reading E1): E ||A h_[S]||^2 = p^2 ||A h||^2 + p(1-p) sum_i
// ||A_i||^2 h_i^2 <= p sum_i (p L + (1-p) ||A_i||^2) h_i^2, with ||A_i||^2 <= ||d_k||^2 for a code
// of filter k, so  tau_k = 1 / (p L_D + (1-p) ||d_k||^2).  tau_used receives tau (eso == 0) or
// tau_k for k = 0..K-1 (eso != 0).
template <typename T>
void code_step(const Dims& D, const T* x, const T* d, T* z, double lam, double step_z, double p,
               uint64_t seed, uint32_t t, double* tau_used, int eso = 0, int mask_mode = 0) {
  std::vector<T> r((size_t)(D.N * D.H * D.W));
  residual<T>(D, x, d, z, r.data());
  const bool per_k = eso != 0 && !(step_z > 0.0);
  std::vector<double> tauk((size_t)D.K);
  if (per_k) {
    const double L = lipschitz_dtft<T>(D, d);
    for (int64_t k = 0; k < D.K; ++k) {
      double dk2 = 0.0;
      for (int64_t a = 0; a < D.s; ++a)
        for (int64_t b = 0; b < D.s; ++b) {
          const double v = (double)d[D.di(k, a, b)];
          dk2 += v * v;
        }
      tauk[k] = (double)(T)(1.0 / (p * L + (1.0 - p) * dk2));
    }
  } else {
    const T tau_t = step_z > 0.0 ? (T)step_z : (T)(1.0 / lipschitz_dtft<T>(D, d));
    for (int64_t k = 0; k < D.K; ++k) tauk[k] = (double)tau_t;
  }
  const uint64_t thr = mask_threshold(p);
  std::vector<double> rd(r.size());
  for (size_t q = 0; q < r.size(); ++q) rd[q] = (double)r[q];
  std::vector<double> dd((size_t)(D.K * D.s * D.s));
  for (size_t q = 0; q < dd.size(); ++q) dd[q] = (double)d[q];
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t k = 0; k < D.K; ++k)
      for (int64_t u = 0; u < D.Hc; ++u)
        for (int64_t v = 0; v < D.Wc; ++v) {
          const uint64_t l = (uint64_t)((k * D.Hc + u) * D.Wc + v);
          if (!mask_bit_mode(mask_mode, seed, t, l, thr)) continue;
          const double c = dtr_at(D, &dd[k * D.s * D.s], &rd[n * D.H * D.W], u, v);
          const int64_t zi = D.zi(n, k, u, v);
          const double w = (double)z[zi] - tauk[k] * c;
          z[zi] = (T)soft_threshold(w, tauk[k] * lam);
        }
  if (tau_used) {
    if (per_k)
      for (int64_t k = 0; k < D.K; ++k) tau_used[k] = tauk[k];
    else
      *tau_used = tauk[0];
  }
}

// ADMM code step (§3.2): Eq.3, the LASSO for the codes
// selected by M^t with the filters held fixed, solved by ADMM with the data term and the L1 term
// split: a quadratic substep solved by Conjugate Gradient ("when N is
// relatively small") and a point-wise shrinkage; 10 iterations, rho = 10 lambda,
// over-relaxation alpha = 1.8.  Readings (A1-A6): scaled form; per image
// (the images are independent problems, Alg.1 lines 5-6); w = y = the current selected codes and
// u = 0 at the start of every outer iteration; CG warm-started at the current w with n_cg
// iterations; the output is the shrunk variable y; unselected codes are untouched (R2).
//   b = x - D z_fix (z_fix: codes with the selected ones zeroed), A = D M^T
//   repeat n_admm:  (A^T A + rho I) w = A^T b + rho (y - u)      [CG]
//                   w^ = alpha w + (1 - alpha) y
//                   y  = S_{lam/rho}(w^ + u),   u = u + w^ - y
template <typename T>
void admm_code_step(const Dims& D, const T* x, const T* d, T* z, double lam, double rho, double alpha,
                    int n_admm, int n_cg, double p, uint64_t seed, uint32_t t) {
  const uint64_t thr = mask_threshold(p);
  const int64_t nc = D.K * D.Hc * D.Wc;
  std::vector<double> dd((size_t)(D.K * D.s * D.s));
  for (size_t q = 0; q < dd.size(); ++q) dd[q] = (double)d[q];
  std::vector<char> msk((size_t)nc);
  for (int64_t l = 0; l < nc; ++l) msk[l] = mask_bit(seed, t, (uint64_t)l, thr) ? 1 : 0;
#pragma omp parallel for schedule(dynamic)
  for (int64_t n = 0; n < D.N; ++n) {
    // image-n views: codes c[l] (l = (k Hc + u) Wc + v), images [i W + j]
    const T* zn = z + n * nc;
    const T* xn = x + n * D.H * D.W;
    // D applied to a code vector (valid true convolution), and D^T at the selected codes
    auto apply_D = [&](const std::vector<double>& c, std::vector<double>& img) {
      for (int64_t i = 0; i < D.H; ++i)
        for (int64_t j = 0; j < D.W; ++j) {
          double acc = 0.0;
          for (int64_t k = 0; k < D.K; ++k)
            for (int64_t a = 0; a < D.s; ++a)
              for (int64_t b = 0; b < D.s; ++b)
                acc += dd[(k * D.s + a) * D.s + b] * c[(k * D.Hc + i + D.P - a) * D.Wc + j + D.P - b];
          img[i * D.W + j] = acc;
        }
    };
    auto apply_Dt_masked = [&](const std::vector<double>& img, std::vector<double>& c) {
      for (int64_t k = 0; k < D.K; ++k)
        for (int64_t u = 0; u < D.Hc; ++u)
          for (int64_t v = 0; v < D.Wc; ++v) {
            const int64_t l = (k * D.Hc + u) * D.Wc + v;
            c[l] = msk[l] ? dtr_at(D, &dd[k * D.s * D.s], img.data(), u, v) : 0.0;
          }
    };
    std::vector<double> zfix((size_t)nc), w((size_t)nc), y((size_t)nc), u((size_t)nc, 0.0);
    for (int64_t l = 0; l < nc; ++l) {
      zfix[l] = msk[l] ? 0.0 : (double)zn[l];
      w[l] = y[l] = msk[l] ? (double)zn[l] : 0.0;
    }
    std::vector<double> img((size_t)(D.H * D.W)), bimg((size_t)(D.H * D.W));
    apply_D(zfix, img);
    for (int64_t q = 0; q < D.H * D.W; ++q) bimg[q] = (double)xn[q] - img[q];  // b = x - D z_fix
    std::vector<double> atb((size_t)nc), r((size_t)nc), pv((size_t)nc), qv((size_t)nc), tmp((size_t)nc);
    apply_Dt_masked(bimg, atb);                                                  // A^T b
    auto apply_op = [&](const std::vector<double>& v, std::vector<double>& out) {  // (A^T A + rho I) v
      apply_D(v, img);
      apply_Dt_masked(img, out);
      for (int64_t l = 0; l < nc; ++l) out[l] = msk[l] ? out[l] + rho * v[l] : 0.0;
    };
    for (int it = 0; it < n_admm; ++it) {
      // CG on (A^T A + rho I) w = A^T b + rho (y - u), warm start at w
      apply_op(w, tmp);
      double rr = 0.0;
      for (int64_t l = 0; l < nc; ++l) {
        r[l] = msk[l] ? atb[l] + rho * (y[l] - u[l]) - tmp[l] : 0.0;
        pv[l] = r[l];
        rr += r[l] * r[l];
      }
      for (int c = 0; c < n_cg && rr > 0.0; ++c) {
        apply_op(pv, qv);
        double pq = 0.0;
        for (int64_t l = 0; l < nc; ++l) pq += pv[l] * qv[l];
        if (!(pq > 0.0)) break;
        const double a = rr / pq;
        double rr2 = 0.0;
        for (int64_t l = 0; l < nc; ++l) {
          w[l] += a * pv[l];
          r[l] -= a * qv[l];
          rr2 += r[l] * r[l];
        }
        const double beta = rr2 / rr;
        for (int64_t l = 0; l < nc; ++l) pv[l] = r[l] + beta * pv[l];
        rr = rr2;
      }
      // over-relaxation, shrinkage, dual update (selected coordinates only)
      for (int64_t l = 0; l < nc; ++l) {
        if (!msk[l]) continue;
        const double wh = alpha * w[l] + (1.0 - alpha) * y[l];
        const double yn = soft_threshold(wh + u[l], lam / rho);
        u[l] += wh - yn;
        y[l] = yn;
      }
    }
    T* zo = z + n * nc;
    for (int64_t l = 0; l < nc; ++l)
      if (msk[l]) zo[l] = (T)y[l];
  }
}

// g[k,a,b] = sum_n sum_{i,j} r[n,i,j] z[n,k,i+P-a,j+P-b]: the gradient of the
// Eq.5 fit term 1/2||x - Z d||^2 with r = Z d - x.
void filter_grad(const Dims& D, const double* r, const double* zd, double* g) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < D.K; ++k)
    for (int64_t a = 0; a < D.s; ++a)
      for (int64_t b = 0; b < D.s; ++b) {
        double acc = 0.0;
        for (int64_t n = 0; n < D.N; ++n)
          for (int64_t i = 0; i < D.H; ++i)
            for (int64_t j = 0; j < D.W; ++j)
              acc += r[(n * D.H + i) * D.W + j] *
                     zd[((n * D.K + k) * D.Hc + i + D.P - a) * D.Wc + j + D.P - b];
        g[D.di(k, a, b)] = acc;
      }
}

// ||Z g||^2 with (Z g)[n,i,j] = sum_k sum_{a,b} g[k,a,b] z[n,k,i+P-a,j+P-b].
double zg_sq(const Dims& D, const double* g, const double* zd) {
  // per-row fp64 partials (rows (n, i) spread over the threads), summed in row order
  std::vector<double> part((size_t)(D.N * D.H), 0.0);
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t i = 0; i < D.H; ++i) {
      double s2 = 0.0;
      for (int64_t j = 0; j < D.W; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < D.K; ++k)
          for (int64_t a = 0; a < D.s; ++a)
            for (int64_t b = 0; b < D.s; ++b)
              acc += g[D.di(k, a, b)] * zd[((n * D.K + k) * D.Hc + i + D.P - a) * D.Wc + j + D.P - b];
        s2 += acc * acc;
      }
      part[n * D.H + i] = s2;
    }
  double tot = 0.0;
  for (size_t q = 0; q < part.size(); ++q) tot += part[q];
  return tot;
}

// One projected-gradient step on the filters (reading R6) for Eq.5 with the
// unit-ball constraint of Eq.1 (reading R7), exact line search (R8).
template <typename T>
void filter_step(const Dims& D, const T* x, T* d, const T* z, double step_d, double* tau_used,
                 double* g_out, double* zg2_out) {
  std::vector<T> rt((size_t)(D.N * D.H * D.W));
  residual<T>(D, x, d, z, rt.data());
  std::vector<double> r(rt.size());
  for (size_t q = 0; q < r.size(); ++q) r[q] = (double)rt[q];
  const size_t nz = (size_t)(D.N * D.K * D.Hc * D.Wc);
  std::vector<double> zd(nz);
  for (size_t q = 0; q < nz; ++q) zd[q] = (double)z[q];
  const size_t nd = (size_t)(D.K * D.s * D.s);
  std::vector<double> g(nd);
  filter_grad(D, r.data(), zd.data(), g.data());
  double tau;
  double zg2 = 0.0;
  if (step_d > 0.0) {
    tau = (double)(T)step_d;
  } else {
    double gg = 0.0;
    for (size_t q = 0; q < nd; ++q) gg += g[q] * g[q];
    zg2 = zg_sq(D, g.data(), zd.data());
    tau = zg2 > 0.0 ? (double)(T)(gg / zg2) : 0.0;
  }
  const int64_t M = D.s * D.s;
  for (int64_t k = 0; k < D.K; ++k) {
    std::vector<double> e((size_t)M);
    double nrm2 = 0.0;
    for (int64_t m = 0; m < M; ++m) {
      e[m] = (double)d[k * M + m] - tau * g[k * M + m];
      nrm2 += e[m] * e[m];
    }
    const double scale = std::max(1.0, std::sqrt(nrm2));
    for (int64_t m = 0; m < M; ++m) d[k * M + m] = (T)(e[m] / scale);
  }
  if (tau_used) *tau_used = tau;
  if (g_out) std::memcpy(g_out, g.data(), nd * sizeof(double));
  if (zg2_out) *zg2_out = zg2;
}

// Projected block-coordinate descent on the filters ("solved
// by projected block coordinate decent ... a single iteration is enough with f computed in previous
// iteration as a warm start"; readings B1-B4).  Blocks = filters, ascending k.  Per block,
// with the other filters fixed, the Eq.5 quadratic in d_k is minimised exactly:
//   C_kk = sum_n Z_nk^T Z_nk (M x M),  g_k = sum_n Z_nk^T r_n (r = Z d - x, current),
//   delta = -(C_kk + eps tr(C_kk)/M I)^{-1} g_k   (Cholesky; eps = BCD_RIDGE, reading B2),
// then d_k <- P_ball(d_k + delta) (R7) and r <- r + Z_k (d_k,new - d_k,old).  tr(C_kk) = 0 (filter k
// has no nonzero code): d_k unchanged, flags[k] = 1.  C, g, r in fp64; d stored in T.
static const double BCD_RIDGE = 1e-10;

// Cholesky factor of the SPD matrix A (n x n, row-major) in place (lower triangle); false if a pivot
// is not positive.
static bool cholesky(std::vector<double>& A, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    double s = A[j * n + j];
    for (int64_t q = 0; q < j; ++q) s -= A[j * n + q] * A[j * n + q];
    if (!(s > 0.0)) return false;
    const double ljj = std::sqrt(s);
    A[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double t = A[i * n + j];
      for (int64_t q = 0; q < j; ++q) t -= A[i * n + q] * A[j * n + q];
      A[i * n + j] = t / ljj;
    }
  }
  return true;
}

template <typename T>
void filter_step_bcd(const Dims& D, const T* x, T* d, const T* z, int sweeps, uint8_t* flags) {
  const int64_t M = D.s * D.s;
  const size_t npx = (size_t)(D.N * D.H * D.W);
  std::vector<double> r(npx);
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t i = 0; i < D.H; ++i)
      for (int64_t j = 0; j < D.W; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < D.K; ++k)
          for (int64_t a = 0; a < D.s; ++a)
            for (int64_t b = 0; b < D.s; ++b)
              acc += (double)d[D.di(k, a, b)] * (double)z[D.zi(n, k, i + D.P - a, j + D.P - b)];
        r[D.xi(n, i, j)] = acc - (double)x[D.xi(n, i, j)];
      }
  if (flags)
    for (int64_t k = 0; k < D.K; ++k) flags[k] = 0;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int64_t k = 0; k < D.K; ++k) {
      std::vector<double> C((size_t)(M * M), 0.0), g((size_t)M, 0.0);
#pragma omp parallel for schedule(static)
      for (int64_t t1 = 0; t1 < M; ++t1) {
        const int64_t a1 = t1 / D.s, b1 = t1 % D.s;
        for (int64_t t2 = 0; t2 < M; ++t2) {
          const int64_t a2 = t2 / D.s, b2 = t2 % D.s;
          double acc = 0.0;
          for (int64_t n = 0; n < D.N; ++n)
            for (int64_t i = 0; i < D.H; ++i)
              for (int64_t j = 0; j < D.W; ++j)
                acc += (double)z[D.zi(n, k, i + D.P - a1, j + D.P - b1)] *
                       (double)z[D.zi(n, k, i + D.P - a2, j + D.P - b2)];
          C[t1 * M + t2] = acc;
        }
        double acc = 0.0;
        for (int64_t n = 0; n < D.N; ++n)
          for (int64_t i = 0; i < D.H; ++i)
            for (int64_t j = 0; j < D.W; ++j)
              acc += r[D.xi(n, i, j)] * (double)z[D.zi(n, k, i + D.P - a1, j + D.P - b1)];
        g[t1] = acc;
      }
      double tr = 0.0;
      for (int64_t m = 0; m < M; ++m) tr += C[m * M + m];
      if (!(tr > 0.0)) {
        if (flags) flags[k] = 1;
        continue;
      }
      const double ridge = BCD_RIDGE * tr / (double)M;
      for (int64_t m = 0; m < M; ++m) C[m * M + m] += ridge;
      if (!cholesky(C, M)) {
        if (flags) flags[k] = 1;
        continue;
      }
      // solve L L^T delta = -g
      std::vector<double> y((size_t)M), e((size_t)M);
      for (int64_t i = 0; i < M; ++i) {
        double t = -g[i];
        for (int64_t q = 0; q < i; ++q) t -= C[i * M + q] * y[q];
        y[i] = t / C[i * M + i];
      }
      for (int64_t i = M - 1; i >= 0; --i) {
        double t = y[i];
        for (int64_t q = i + 1; q < M; ++q) t -= C[q * M + i] * e[q];
        e[i] = t / C[i * M + i];
      }
      double nrm2 = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        e[m] += (double)d[k * M + m];
        nrm2 += e[m] * e[m];
      }
      const double scale = std::max(1.0, std::sqrt(nrm2));
      std::vector<double> dl((size_t)M);
      for (int64_t m = 0; m < M; ++m) {
        const T dn = (T)(e[m] / scale);
        dl[m] = (double)dn - (double)d[k * M + m];
        d[k * M + m] = dn;
      }
#pragma omp parallel for schedule(static)
      for (int64_t n = 0; n < D.N; ++n)
        for (int64_t i = 0; i < D.H; ++i)
          for (int64_t j = 0; j < D.W; ++j) {
            double acc = 0.0;
            for (int64_t a = 0; a < D.s; ++a)
              for (int64_t b = 0; b < D.s; ++b)
                acc += dl[a * D.s + b] * (double)z[D.zi(n, k, i + D.P - a, j + D.P - b)];
            r[D.xi(n, i, j)] += acc;
          }
    }
}

// Online surrogates (§3.3, Eq.7): after the t-th
// mini-batch (codes z, images x),
//   C^t = ((t-1)/t) C^{t-1} + (1/t) sum_n Z_n^T Z_n,   B^t = ((t-1)/t) B^{t-1} + (1/t) sum_n Z_n^T x_n,
// C stored block-major [K][K][M][M] (block (k1,k2), entry (t1,t2) = sum z_k1[p-t1] z_k2[p-t2]),
// B [K][M].  t is the count after the update (t >= 1).  fp64 throughout.
template <typename T>
void surrogate_update(const Dims& D, const T* x, const T* z, double* C, double* B, int64_t t) {
  const int64_t M = D.s * D.s, K = D.K;
  const double wo = (double)(t - 1) / (double)t, wn = 1.0 / (double)t;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t k1 = 0; k1 < K; ++k1)
    for (int64_t t1 = 0; t1 < M; ++t1) {
      const int64_t a1 = t1 / D.s, b1 = t1 % D.s;
      for (int64_t k2 = 0; k2 < K; ++k2)
        for (int64_t t2 = 0; t2 < M; ++t2) {
          const int64_t a2 = t2 / D.s, b2 = t2 % D.s;
          double acc = 0.0;
          for (int64_t n = 0; n < D.N; ++n)
            for (int64_t i = 0; i < D.H; ++i)
              for (int64_t j = 0; j < D.W; ++j)
                acc += (double)z[D.zi(n, k1, i + D.P - a1, j + D.P - b1)] *
                       (double)z[D.zi(n, k2, i + D.P - a2, j + D.P - b2)];
          double& c = C[((k1 * K + k2) * M + t1) * M + t2];
          c = wo * c + wn * acc;
        }
      double acc = 0.0;
      for (int64_t n = 0; n < D.N; ++n)
        for (int64_t i = 0; i < D.H; ++i)
          for (int64_t j = 0; j < D.W; ++j)
            acc += (double)x[D.xi(n, i, j)] * (double)z[D.zi(n, k1, i + D.P - a1, j + D.P - b1)];
      B[k1 * M + t1] = wo * B[k1 * M + t1] + wn * acc;
    }
}

// Eq.8: min_d 1/2 d^T C d - d^T B  s.t. ||d_k|| <= 1, by the projected block-coordinate
// sweep of filter_step_bcd with the surrogate in place of the data: per k in order,
//   g_k = sum_k' C_kk' d_k' - B_k,  d_k <- P_ball(d_k - (C_kk + eps tr(C_kk)/M I)^-1 g_k).
// tr(C_kk) = 0: unchanged, flags[k] = 1.
template <typename T>
void filter_step_surrogate(int64_t K, int64_t s, const double* C, const double* B, T* d, int sweeps,
                           uint8_t* flags) {
  const int64_t M = s * s;
  if (flags)
    for (int64_t k = 0; k < K; ++k) flags[k] = 0;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int64_t k = 0; k < K; ++k) {
      std::vector<double> A((size_t)(M * M)), g((size_t)M);
      for (int64_t t1 = 0; t1 < M; ++t1) {
        double acc = -B[k * M + t1];
        for (int64_t k2 = 0; k2 < K; ++k2)
          for (int64_t t2 = 0; t2 < M; ++t2) acc += C[((k * K + k2) * M + t1) * M + t2] * (double)d[k2 * M + t2];
        g[t1] = acc;
        for (int64_t t2 = 0; t2 < M; ++t2) A[t1 * M + t2] = C[((k * K + k) * M + t1) * M + t2];
      }
      double tr = 0.0;
      for (int64_t m = 0; m < M; ++m) tr += A[m * M + m];
      if (!(tr > 0.0)) {
        if (flags) flags[k] = 1;
        continue;
      }
      for (int64_t m = 0; m < M; ++m) A[m * M + m] += BCD_RIDGE * tr / (double)M;
      if (!cholesky(A, M)) {
        if (flags) flags[k] = 1;
        continue;
      }
      std::vector<double> y((size_t)M), e((size_t)M);
      for (int64_t i = 0; i < M; ++i) {
        double tt = -g[i];
        for (int64_t q = 0; q < i; ++q) tt -= A[i * M + q] * y[q];
        y[i] = tt / A[i * M + i];
      }
      for (int64_t i = M - 1; i >= 0; --i) {
        double tt = y[i];
        for (int64_t q = i + 1; q < M; ++q) tt -= A[q * M + i] * e[q];
        e[i] = tt / A[i * M + i];
      }
      double nrm2 = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        e[m] += (double)d[k * M + m];
        nrm2 += e[m] * e[m];
      }
      const double scale = std::max(1.0, std::sqrt(nrm2));
      for (int64_t m = 0; m < M; ++m) d[k * M + m] = (T)(e[m] / scale);
    }
}

// Eq.1 objective: F = sum_n 1/2||x_n - sum_k d_k * z_{n,k}||^2 + lam sum ||z||_1.
template <typename T>
void objective(const Dims& D, const T* x, const T* d, const T* z, double lam, double out[3]) {
  // per-row fp64 partials of the squared residual (rows (n, i) spread over the threads) and per-image
  // partials of |z|, each summed in a fixed order
  std::vector<double> h((size_t)(D.N * D.H), 0.0), l1((size_t)D.N, 0.0);
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < D.N; ++n)
    for (int64_t i = 0; i < D.H; ++i) {
      double s2 = 0.0;
      for (int64_t j = 0; j < D.W; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < D.K; ++k)
          for (int64_t a = 0; a < D.s; ++a)
            for (int64_t b = 0; b < D.s; ++b)
              acc += (double)d[D.di(k, a, b)] * (double)z[D.zi(n, k, i + D.P - a, j + D.P - b)];
        const double rr = acc - (double)x[D.xi(n, i, j)];
        s2 += rr * rr;
      }
      h[n * D.H + i] = s2;
    }
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < D.N; ++n) {
    double a1 = 0.0;
    for (int64_t k = 0; k < D.K; ++k)
      for (int64_t u = 0; u < D.Hc; ++u)
        for (int64_t v = 0; v < D.Wc; ++v) a1 += std::fabs((double)z[D.zi(n, k, u, v)]);
    l1[n] = a1;
  }
  double hs = 0.0, ls = 0.0;
  for (size_t q = 0; q < h.size(); ++q) hs += h[q];
  hs *= 0.5;
  for (int64_t n = 0; n < D.N; ++n) ls += l1[n];
  out[1] = hs;
  out[2] = lam * ls;
  out[0] = out[1] + out[2];
}

}  // namespace

// ---------------------------------------------------------------------------
// C interface (ctypes).  All pointers are host pointers to contiguous arrays:
// x[N][H][W], d[K][s][s], z[N][K][H+s-1][W+s-1], r[N][H][W].
// ---------------------------------------------------------------------------
extern "C" {

int oracle_num_threads() { return omp_get_max_threads(); }

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox4x32_10(ctr, key, out);
}

void oracle_philox_batch(int64_t count, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  for (int64_t q = 0; q < count; ++q) philox4x32_10(ctr + 4 * q, key + 2 * q, out + 4 * q);
}

uint64_t oracle_mask_threshold(double p) { return mask_threshold(p); }

// Mask bits in the ABI layout: bit l of word l>>5 (LSB first).
void oracle_mask_bits_mode(int64_t K, int64_t Hc, int64_t Wc, double p, uint64_t seed, uint32_t t,
                           uint32_t* bits, int mode) {
  const uint64_t total = (uint64_t)(K * Hc * Wc);
  const uint64_t nwords = (total + 31) / 32;
  const uint64_t thr = mask_threshold(p);
#pragma omp parallel for schedule(static)
  for (int64_t wi = 0; wi < (int64_t)nwords; ++wi) {
    uint32_t word = 0;
    for (uint64_t bit = 0; bit < 32; ++bit) {
      const uint64_t l = (uint64_t)wi * 32 + bit;
      if (l < total && mask_bit_mode(mode, seed, t, l, thr)) word |= (1u << bit);
    }
    bits[wi] = word;
  }
}

void oracle_mask_bits(int64_t K, int64_t Hc, int64_t Wc, double p, uint64_t seed, uint32_t t,
                      uint32_t* bits) {
  const uint64_t total = (uint64_t)(K * Hc * Wc);
  const uint64_t nwords = (total + 31) / 32;
  const uint64_t thr = mask_threshold(p);
#pragma omp parallel for schedule(static)
  for (int64_t wi = 0; wi < (int64_t)nwords; ++wi) {
    uint32_t word = 0;
    for (uint64_t bit = 0; bit < 32; ++bit) {
      const uint64_t l = (uint64_t)wi * 32 + bit;
      if (l < total && mask_bit(seed, t, l, thr)) word |= (1u << bit);
    }
    bits[wi] = word;
  }
}

double oracle_soft_threshold(double w, double kappa) { return soft_threshold(w, kappa); }

#define ORACLE_EXPORTS(T, SUF)                                                                    \
  void oracle_residual_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W, const T* x,  \
                             const T* d, const T* z, T* r) {                                     \
    residual<T>(Dims(N, K, s, H, W), x, d, z, r);                                                \
  }                                                                                              \
  void oracle_dtr_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W, const T* d,       \
                        const T* r, T* out) {                                                    \
    dtr_all<T>(Dims(N, K, s, H, W), d, r, out);                                                  \
  }                                                                                              \
  void oracle_filter_grad_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W,           \
                                const T* r, const T* z, double* g) {                             \
    Dims D(N, K, s, H, W);                                                                       \
    std::vector<double> rd((size_t)(N * H * W)), zd((size_t)(N * K * D.Hc * D.Wc));              \
    for (size_t q = 0; q < rd.size(); ++q) rd[q] = (double)r[q];                                  \
    for (size_t q = 0; q < zd.size(); ++q) zd[q] = (double)z[q];                                  \
    filter_grad(D, rd.data(), zd.data(), g);                                                     \
  }                                                                                              \
  double oracle_lipschitz_##SUF(int64_t K, int64_t s, const T* d) {                              \
    return lipschitz_dtft<T>(Dims(1, K, s, s, s), d);                                            \
  }                                                                                              \
  void oracle_code_step_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W, const T* x, \
                              const T* d, T* z, double lam, double step_z, double p,             \
                              uint64_t seed, uint32_t t, double* tau_used, int eso, int mmode) { \
    code_step<T>(Dims(N, K, s, H, W), x, d, z, lam, step_z, p, seed, t, tau_used, eso, mmode);  \
  }                                                                                              \
  void oracle_admm_code_step_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W,          \
                                   const T* x, const T* d, T* z, double lam, double rho,           \
                                   double alpha, int n_admm, int n_cg, double p, uint64_t seed,    \
                                   uint32_t t) {                                                   \
    admm_code_step<T>(Dims(N, K, s, H, W), x, d, z, lam, rho, alpha, n_admm, n_cg, p, seed, t);   \
  }                                                                                              \
  void oracle_filter_step_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W,           \
                                const T* x, T* d, const T* z, double step_d, double* tau_used,   \
                                double* g_out, double* zg2_out) {                                \
    filter_step<T>(Dims(N, K, s, H, W), x, d, z, step_d, tau_used, g_out, zg2_out);             \
  }                                                                                              \
  void oracle_filter_step_bcd_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W,       \
                                    const T* x, T* d, const T* z, int sweeps, uint8_t* flags) {    \
    filter_step_bcd<T>(Dims(N, K, s, H, W), x, d, z, sweeps, flags);                             \
  }                                                                                              \
  void oracle_surrogate_update_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W,      \
                                     const T* x, const T* z, double* C, double* B, int64_t t) {    \
    surrogate_update<T>(Dims(N, K, s, H, W), x, z, C, B, t);                                     \
  }                                                                                              \
  void oracle_filter_step_surrogate_##SUF(int64_t K, int64_t s, const double* C, const double* B,  \
                                          T* d, int sweeps, uint8_t* flags) {                    \
    filter_step_surrogate<T>(K, s, C, B, d, sweeps, flags);                                      \
  }                                                                                              \
  void oracle_objective_##SUF(int64_t N, int64_t K, int64_t s, int64_t H, int64_t W, const T* x, \
                              const T* d, const T* z, double lam, double out[3]) {               \
    objective<T>(Dims(N, K, s, H, W), x, d, z, lam, out);                                        \
  }

ORACLE_EXPORTS(float, f32)
ORACLE_EXPORTS(double, f64)

}  // extern "C"

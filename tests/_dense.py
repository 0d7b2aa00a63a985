"""Dense-matrix brute force for tiny CSC instances (test helper, no oracle code).

The convolution "*" of Eq.1 is taken from scipy's
convolve2d in 'valid' mode (reading R3: codes are (H+s-1)x(W+s-1), the output
is H x W with no wrap-around).  The Toeplitz matrices D and Z
 are materialised column by column as impulse responses of that
library routine, so nothing here re-types the oracle's index arithmetic.
"""
import numpy as np
from scipy.signal import convolve2d


def conv_valid(z2d, f2d):
    return convolve2d(z2d, f2d, mode="valid")


def dense_D(d, H, W):
    """A = [D_1 .. D_K] in R^{HW x K*Hc*Wc}: A @ vec(z_n) = vec(sum_k d_k * z_{n,k})."""
    K, s, _ = d.shape
    Hc, Wc = H + s - 1, W + s - 1
    A = np.zeros((H * W, K * Hc * Wc))
    col = 0
    for k in range(K):
        for u in range(Hc):
            for v in range(Wc):
                e = np.zeros((Hc, Wc))
                e[u, v] = 1.0
                A[:, col] = conv_valid(e, d[k].astype(np.float64)).ravel()
                col += 1
    return A


def dense_Z(z_n, s):
    """Z in R^{HW x K*s*s} for one image: Z @ vec(d) = vec(sum_k d_k * z_{n,k})."""
    K, Hc, Wc = z_n.shape
    H, W = Hc - s + 1, Wc - s + 1
    Z = np.zeros((H * W, K * s * s))
    col = 0
    for k in range(K):
        for a in range(s):
            for b in range(s):
                e = np.zeros((s, s))
                e[a, b] = 1.0
                Z[:, col] = conv_valid(z_n[k].astype(np.float64), e).ravel()
                col += 1
    return Z


def recon(d, z):
    """sum_k d_k * z_{n,k} for all n via scipy (fp64)."""
    N, K = z.shape[:2]
    out = []
    for n in range(N):
        acc = None
        for k in range(K):
            c = conv_valid(z[n, k].astype(np.float64), d[k].astype(np.float64))
            acc = c if acc is None else acc + c
        out.append(acc)
    return np.stack(out)


def soft(w, kappa):
    return np.sign(w) * np.maximum(np.abs(w) - kappa, 0.0)

"""Pins of the oracle's ADMM code solver (§3.2).

The operator of the LASSO (Eq.3) is materialised independently of the oracle: tests/_dense.py
builds D from scipy impulse responses.  The pins:
  * at p = 1 and with enough ADMM / CG iterations the oracle reaches the LASSO minimiser found by a
    long accelerated proximal-gradient run on the dense matrix (a different algorithm);
  * at p < 1 the result satisfies the LASSO optimality (KKT) conditions on the selected codes and
    leaves the other codes untouched;
  * lambda >= ||A^T b||_inf drives the codes to the minimiser 0;
  * one oracle step equals the same ADMM/CG sequence run with the dense matrix (fp64).
"""
import numpy as np
import pytest

import oracle
from tests._dense import dense_D, soft


def _problem(seed, K=2, s=3, H=5, W=6):
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((K, s, s))
    d /= np.sqrt((d ** 2).sum(axis=(1, 2), keepdims=True))
    x = rng.standard_normal((1, H, W))
    z = np.zeros((1, K, H + s - 1, W + s - 1))
    return x, d, z


def _fista(A, b, lam, iters=20000):
    L = np.linalg.norm(A, 2) ** 2
    w = np.zeros(A.shape[1]); yk = w.copy(); tk = 1.0
    for _ in range(iters):
        w_new = soft(yk - A.T @ (A @ yk - b) / L, lam / L)
        t_new = 0.5 * (1 + np.sqrt(1 + 4 * tk * tk))
        yk = w_new + (tk - 1) / t_new * (w_new - w)
        w, tk = w_new, t_new
    return w


def test_admm_reaches_lasso_minimiser_at_p1():
    """The LASSO value reached by ADMM (p = 1: every code selected, M = I) equals the
    minimum found by FISTA on the dense matrix, and the minimisers agree."""
    x, d, z = _problem(1)
    lam = 0.3
    A = dense_D(d, 5, 6)
    b = x.ravel()
    w_ref = _fista(A, b, lam, iters=60000)
    zo = oracle.admm_code_step(x, d, z, lam, 1.0, 7, 1, n_admm=3000, n_cg=60, dtype=np.float64).ravel()
    f = lambda w: 0.5 * np.sum((A @ w - b) ** 2) + lam * np.abs(w).sum()
    assert abs(f(zo) - f(w_ref)) <= 1e-9 * f(w_ref), (f(zo), f(w_ref))
    err = np.linalg.norm(zo - w_ref) / np.linalg.norm(w_ref)
    assert np.linalg.norm(w_ref) > 0 and err < 1e-4, err


@pytest.mark.parametrize("p", [0.5, 0.2])
def test_admm_kkt_on_selected_codes(p):
    x, d, z0 = _problem(2)
    rng = np.random.default_rng(3)
    z0 = rng.standard_normal(z0.shape) * (rng.random(z0.shape) < 0.4)
    lam, seed, t = 0.2, 99, 4
    zo = oracle.admm_code_step(x, d, z0, lam, p, seed, t, n_admm=3000, n_cg=60, dtype=np.float64)
    K, Hc, Wc = z0.shape[1:]
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, t), K, Hc, Wc).ravel()
    assert m.any() and (~m).any()
    assert np.array_equal(zo.ravel()[~m], z0.ravel()[~m])  # unselected codes untouched (R2)
    A = dense_D(d, 5, 6)
    g = A[:, m].T @ (x.ravel() - A @ zo.ravel())           # -gradient of the fit term on M
    ym = zo.ravel()[m]
    nz = np.abs(ym) > 1e-9
    assert np.allclose(g[nz], lam * np.sign(ym[nz]), atol=1e-6)
    assert (np.abs(g[~nz]) <= lam + 1e-6).all()


def test_admm_large_lambda_keeps_zero_codes():
    x, d, z = _problem(4)
    A = dense_D(d, 5, 6)
    lam = 1.01 * np.abs(A.T @ x.ravel()).max()
    zo = oracle.admm_code_step(x, d, z, lam, 1.0, 5, 2, n_admm=2000, n_cg=60, dtype=np.float64)
    assert np.abs(zo).max() <= 1e-9


def test_admm_step_equals_dense_matrix_run():
    """One oracle step (10 ADMM iterations, 5 CG iterations, rho = 10 lambda, alpha = 1.8) equals the
    same sequence on the dense operator: checks the oracle's matrix-free D / D^T and masking."""
    x, d, z0 = _problem(5, K=3, H=6, W=5)
    rng = np.random.default_rng(6)
    z0 = rng.standard_normal(z0.shape) * (rng.random(z0.shape) < 0.5)
    lam, p, seed, t = 0.25, 0.5, 1234, 9
    rho, alpha = 10 * lam, 1.8
    zo = oracle.admm_code_step(x, d, z0, lam, p, seed, t, dtype=np.float64)
    K, Hc, Wc = z0.shape[1:]
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, t), K, Hc, Wc).ravel()
    A = dense_D(d, 6, 5)
    Am = A[:, m]
    zf = z0.ravel().copy()
    zf[m] = 0.0
    b = x.ravel() - A @ zf
    w = z0.ravel()[m].copy(); y = w.copy(); u = np.zeros_like(w)
    Q = Am.T @ Am + rho * np.eye(Am.shape[1])
    atb = Am.T @ b
    for _ in range(oracle.ADMM_ITERS):
        r = atb + rho * (y - u) - Q @ w
        pv = r.copy(); rr = r @ r
        for _ in range(oracle.ADMM_CG_ITERS):
            if rr <= 0:
                break
            q = Q @ pv
            a = rr / (pv @ q)
            w = w + a * pv
            r = r - a * q
            rr2 = r @ r
            pv = r + (rr2 / rr) * pv
            rr = rr2
        wh = alpha * w + (1 - alpha) * y
        yn = soft(wh + u, lam / rho)
        u = u + wh - yn
        y = yn
    ref = z0.ravel().copy()
    ref[m] = y
    assert np.abs(zo.ravel() - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())

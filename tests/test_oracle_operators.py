"""Pins of the oracle's operators: D z, D^T r (gradient of the
Eq.3 fit term), Z^T r (gradient of the Eq.5 fit term) and the
Eq.1 objective.

Pins: scipy convolve2d/correlate2d (library routines), dense Toeplitz
brute force built from impulse responses, the adjoint identities in the fp64
oracle build, finite differences, the impulse response and no-wrap boundary, and
the objective's closed-form special cases.
"""
import numpy as np
import pytest
from scipy.signal import correlate2d

import oracle
from synth import random_problem
from tests._dense import conv_valid, dense_D, dense_Z, recon
from tests.conftest import rel_err


@pytest.mark.parametrize("shape", [(2, 3, 3, 6, 7), (1, 2, 5, 9, 8), (2, 1, 1, 4, 4)])
def test_residual_matches_scipy_valid_convolution(shape):
    N, K, s, H, W = shape
    x, d, z = random_problem(1, N, K, s, H, W, dtype=np.float64)
    r = oracle.residual(x, d, z, dtype=np.float64)
    ref = recon(d, z) - x
    assert rel_err(r, ref) < 1e-13


def test_residual_matches_dense_toeplitz():
    N, K, s, H, W = 2, 2, 3, 5, 6
    x, d, z = random_problem(2, N, K, s, H, W, dtype=np.float64)
    A = dense_D(d, H, W)
    r = oracle.residual(x, d, z, dtype=np.float64)
    for n in range(N):
        ref = A @ z[n].ravel() - x[n].ravel()
        assert rel_err(r[n].ravel(), ref) < 1e-13


def test_residual_f32_state_close_to_f64():
    x, d, z = random_problem(3, 2, 4, 5, 12, 10, dtype=np.float32)
    r32 = oracle.residual(x, d, z, dtype=np.float32)
    r64 = oracle.residual(x, d, z, dtype=np.float64)
    assert r32.dtype == np.float32
    assert rel_err(r32, r64) < 1e-6


def test_impulse_response_and_no_wrap():
    """A unit code at (u,v) reproduces d_k at offset (u-P, v-P), truncated at the border."""
    K, s, H, W = 1, 3, 6, 6
    P = s - 1
    d = np.arange(1, 10, dtype=np.float64).reshape(1, 3, 3)
    Hc = H + P
    z = np.zeros((1, K, Hc, Hc))
    z[0, 0, 4, 5] = 1.0
    r = oracle.residual(None, d, z, dtype=np.float64)[0]
    expect = np.zeros((H, W))
    for a in range(s):
        for b in range(s):
            i, j = 4 - P + a, 5 - P + b
            if 0 <= i < H and 0 <= j < W:
                expect[i, j] = d[0, a, b]
    assert np.array_equal(r, expect)
    # corner impulse: only r[0,0] = d[P,P], nothing wraps to the far corner
    z[:] = 0
    z[0, 0, 0, 0] = 1.0
    r = oracle.residual(None, d, z, dtype=np.float64)[0]
    assert r[0, 0] == d[0, P, P]
    assert np.count_nonzero(r) == 1 and r[H - 1, W - 1] == 0.0


def test_zero_codes_give_minus_x():
    x, d, z = random_problem(4, 2, 3, 3, 5, 5, dtype=np.float32)
    r = oracle.residual(x, d, np.zeros_like(z), dtype=np.float32)
    assert np.array_equal(r, -x)


@pytest.mark.parametrize("shape", [(2, 3, 3, 6, 7), (1, 2, 5, 8, 9)])
def test_dtr_matches_scipy_full_correlation(shape):
    N, K, s, H, W = shape
    _, d, _ = random_problem(5, N, K, s, H, W, dtype=np.float64)
    r = np.random.default_rng(5).standard_normal((N, H, W))
    g = oracle.dtr(d, r, dtype=np.float64)
    for n in range(N):
        for k in range(K):
            ref = correlate2d(r[n], d[k], mode="full")
            assert rel_err(g[n, k], ref) < 1e-13


def test_adjoint_identity_D():
    """<D z, r> = <z, D^T r> in the fp64 oracle build."""
    for seed in range(5):
        N, K, s, H, W = 2, 3, [1, 3, 5][seed % 3], 9 + seed, 7 + seed
        _, d, z = random_problem(10 + seed, N, K, s, H, W, dtype=np.float64)
        rr = np.random.default_rng(seed).standard_normal((N, H, W))
        lhs = np.vdot(oracle.residual(None, d, z, dtype=np.float64), rr)
        rhs = np.vdot(z, oracle.dtr(d, rr, dtype=np.float64))
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(z) * np.linalg.norm(rr) * np.sqrt(K * s * s)


def test_filter_grad_matches_scipy_and_adjoint_Z():
    N, K, s, H, W = 2, 3, 5, 9, 8
    _, d, z = random_problem(20, N, K, s, H, W, dtype=np.float64)
    rr = np.random.default_rng(20).standard_normal((N, H, W))
    g = oracle.filter_grad(rr, z, dtype=np.float64)
    ref = np.zeros_like(g)
    for n in range(N):
        for k in range(K):
            ref[k] += correlate2d(z[n, k], rr[n], mode="valid")[::-1, ::-1]
    assert rel_err(g, ref) < 1e-13
    # <Z d, r> = <d, Z^T r>
    lhs = np.vdot(oracle.residual(None, d, z, dtype=np.float64), rr)
    rhs = np.vdot(d, g)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs) + 1e-12
    # dense Z brute force
    for n in range(N):
        Zm = dense_Z(z[n], s)
        assert rel_err(Zm @ d.ravel(), oracle.residual(None, d, z[n:n + 1], dtype=np.float64).ravel()) < 1e-13


def test_filter_grad_finite_differences():
    """g is the gradient of f(d) = 1/2||sum_k d_k*z_k - x||^2 (central differences, exact for a quadratic)."""
    N, K, s, H, W = 1, 2, 3, 6, 5
    x, d, z = random_problem(21, N, K, s, H, W, dtype=np.float64)
    r = oracle.residual(x, d, z, dtype=np.float64)
    g = oracle.filter_grad(r, z, dtype=np.float64)

    def f(dd):
        return 0.5 * np.sum((recon(dd, z) - x) ** 2)

    h = 1e-3
    fd = np.zeros_like(d)
    for idx in np.ndindex(d.shape):
        e = np.zeros_like(d)
        e[idx] = h
        fd[idx] = (f(d + e) - f(d - e)) / (2 * h)
    assert rel_err(g, fd) < 1e-8


def test_objective_special_cases():
    N, K, s, H, W = 2, 3, 3, 7, 6
    x, d, z = random_problem(30, N, K, s, H, W, dtype=np.float64)
    # zero codes -> 1/2 sum ||x||^2
    F, fit, l1 = oracle.objective(x, d, np.zeros_like(z), 1.0, dtype=np.float64)
    assert abs(F - 0.5 * np.sum(x * x)) < 1e-12 * F and l1 == 0.0
    # perfect fit, lambda = 0 -> 0
    xf = recon(d, z)
    F, fit, l1 = oracle.objective(xf, d, z, 0.0, dtype=np.float64)
    assert F < 1e-20 * np.sum(xf * xf) + 1e-24
    # dense evaluation
    lam = 0.7
    A = dense_D(d, H, W)
    ref = sum(0.5 * np.sum((A @ z[n].ravel() - x[n].ravel()) ** 2) for n in range(N)) + lam * np.abs(z).sum()
    F, fit, l1 = oracle.objective(x, d, z, lam, dtype=np.float64)
    assert abs(F - ref) < 1e-12 * ref
    assert abs(F - fit - l1) < 1e-12 * F

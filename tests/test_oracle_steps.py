"""Pins of the oracle's iteration steps.

a3 code step (Eq.3-4, readings R1/R2): at p=1 it is exactly
the textbook ISTA step z+ = S_{tau*lam}(z - tau*A^T(Az - x)) with the dense
Toeplitz A; at p<1 the same step restricted to the masked columns with every
other code bit-identical; monotone for tau <= 1/L; lam >= ||A^T x||_inf keeps
z = 0.  Shrinkage closed forms and prox optimality.
a5 filter step (Eq.5 + unit ball, readings R6-R8): the
line-search step is the exact minimiser of the 1-D quadratic; the projection
bound; zero codes leave d unchanged.
a7 Lipschitz bound (reading R8): delta filter -> 1; equals the numpy FFT of the
zero-padded filters on the 64x64 grid; bounds ||A||_2^2 on small domains.
"""
import numpy as np
import pytest

import oracle
from synth import random_problem, CONFIGS, make_filters, make_images, make_codes, mask_seed
from tests._dense import dense_D, dense_Z, recon, soft
from tests.conftest import rel_err


def test_soft_threshold_closed_forms():
    assert oracle.soft_threshold(2.0, 0.5) == 1.5
    assert oracle.soft_threshold(-0.3, 0.5) == 0.0
    assert oracle.soft_threshold(-2.0, 0.5) == -1.5
    assert oracle.soft_threshold(0.0, 0.0) == 0.0
    # +0.0 for the thresholded zone (reading #12)
    assert np.copysign(1.0, oracle.soft_threshold(-0.3, 0.5)) == 1.0


def test_soft_threshold_is_prox_of_l1():
    """u = S(v,k) minimises 1/2(u-v)^2 + k|u|: v - u in k * subdiff|u| (subgradient check)."""
    rng = np.random.default_rng(0)
    for v, k in zip(rng.standard_normal(200) * 3, rng.random(200) * 2):
        u = oracle.soft_threshold(v, k)
        if u != 0.0:
            assert abs((v - u) - k * np.sign(u)) < 1e-12
        else:
            assert abs(v) <= k + 1e-15
        for du in (-1e-3, 1e-3):
            assert 0.5 * (u - v) ** 2 + k * abs(u) <= 0.5 * (u + du - v) ** 2 + k * abs(u + du) + 1e-15


def _dense_stack(d, H, W):
    return dense_D(d, H, W)


@pytest.mark.parametrize("p", [1.0, 0.5, 0.2])
def test_code_step_is_masked_textbook_ista(p):
    N, K, s, H, W = 2, 2, 3, 5, 6
    x, d, z = random_problem(40, N, K, s, H, W, code_density=0.5, dtype=np.float64)
    lam, tau, seed, t = 0.3, 0.05, 77, 4
    A = _dense_stack(d, H, W)
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, t), K, Hc, Wc).ravel()
    if p == 1.0:
        assert m.all()
    z1, tau_used = oracle.code_step(x, d, z, lam, tau, p, seed, t, dtype=np.float64)
    assert tau_used == tau
    for n in range(N):
        zn = z[n].ravel()
        grad = A.T @ (A @ zn - x[n].ravel())
        ista = soft(zn - tau * grad, tau * lam)
        expect = np.where(m, ista, zn)
        assert rel_err(z1[n].ravel(), expect) < 1e-13
        # unmasked codes are bit-identical
        assert np.array_equal(z1[n].ravel()[~m], zn[~m])


def test_code_step_f32_unmasked_bit_identical():
    x, d, z = random_problem(41, 2, 3, 5, 9, 8, code_density=0.3, dtype=np.float32)
    Hc, Wc = z.shape[2:]
    m = oracle.unpack_mask(oracle.mask_bits(3, Hc, Wc, 0.1, 5, 9), 3, Hc, Wc)
    z1, _ = oracle.code_step(x, d, z, 1.0, 0.0, 0.1, 5, 9, dtype=np.float32)
    assert z1.dtype == np.float32
    for n in range(2):
        assert np.array_equal(z1[n][~m], z[n][~m])


def test_code_step_default_tau_is_inverse_lipschitz():
    x, d, z = random_problem(42, 1, 3, 5, 8, 8, dtype=np.float32)
    _, tau = oracle.code_step(x, d, z, 1.0, 0.0, 0.5, 1, 1, dtype=np.float32)
    L = oracle.lipschitz(d, dtype=np.float32)
    assert tau == float(np.float32(1.0 / L))


@pytest.mark.parametrize("p", [1.0, 0.3])
def test_code_step_monotone_with_step_1_over_L(p):
    N, K, s, H, W = 1, 3, 3, 6, 6
    x, d, z = random_problem(43, N, K, s, H, W, code_density=0.4, dtype=np.float64)
    A = _dense_stack(d, H, W)
    L = np.linalg.norm(A, 2) ** 2
    lam = 0.2
    F0 = oracle.objective(x, d, z, lam, dtype=np.float64)[0]
    zz = z
    for t in range(1, 30):
        zz, _ = oracle.code_step(x, d, zz, lam, 1.0 / L, p, 3, t, dtype=np.float64)
        F1 = oracle.objective(x, d, zz, lam, dtype=np.float64)[0]
        assert F1 <= F0 + 1e-12 * abs(F0)
        F0 = F1


def test_large_lambda_keeps_codes_zero():
    N, K, s, H, W = 2, 3, 3, 7, 7
    x, d, _ = random_problem(44, N, K, s, H, W, dtype=np.float64)
    z0 = np.zeros((N, K, H + s - 1, W + s - 1))
    A = _dense_stack(d, H, W)
    tau = 1.0 / (np.linalg.norm(A, 2) ** 2)
    lam = max(np.abs(A.T @ x[n].ravel()).max() for n in range(N)) * 1.0001
    z1, _ = oracle.code_step(x, d, z0, lam, tau, 1.0, 1, 1, dtype=np.float64)
    assert not z1.any()


def test_lipschitz_delta_filter_is_one():
    d = np.zeros((1, 5, 5), dtype=np.float32)
    d[0, 2, 2] = 1.0
    assert abs(oracle.lipschitz(d, dtype=np.float32) - 1.0) < 4e-16  # |e^{i theta}|^2 = 1 up to cos/sin rounding
    d[0, 2, 2] = 0.0
    d[0, 0, 4] = 1.0  # a shifted delta has the same magnitude response
    assert abs(oracle.lipschitz(d, dtype=np.float64) - 1.0) < 1e-12


def test_lipschitz_matches_numpy_fft_grid():
    d = make_filters(CONFIGS["tiny"]).astype(np.float64)
    L = oracle.lipschitz(d, dtype=np.float64)
    spec = np.abs(np.fft.fft2(d, s=(64, 64))) ** 2
    assert abs(L - spec.sum(axis=0).max()) < 1e-12 * L


def test_lipschitz_bounds_operator_norm_on_small_domains():
    for seed, (K, s, H) in enumerate([(3, 3, 6), (2, 5, 8), (4, 3, 5)]):
        _, d, _ = random_problem(50 + seed, 1, K, s, H, H, dtype=np.float64)
        A = _dense_stack(d, H, H)
        assert oracle.lipschitz(d, dtype=np.float64) >= np.linalg.norm(A, 2) ** 2 * (1 - 1e-9)


def test_filter_step_line_search_is_exact_minimiser():
    N, K, s, H, W = 2, 3, 3, 7, 6
    x, d, z = random_problem(60, N, K, s, H, W, code_density=0.6, dtype=np.float64)
    d_new, tau, g, zg2 = oracle.filter_step(x, d, z, 0.0, dtype=np.float64)

    def f(tt):  # fit term along the ray d - tt*g (before projection)
        return 0.5 * np.sum((recon(d - tt * g, z) - x) ** 2)

    # the exact minimiser of the 1-D quadratic from three evaluations (no oracle formula involved)
    h = tau
    f0, f1, f2 = f(0.0), f(h), f(2 * h)
    curv = (f2 - 2 * f1 + f0) / (h * h)
    slope0 = (4 * f1 - 3 * f0 - f2) / (2 * h)
    assert abs(tau - (-slope0 / curv)) < 1e-8 * tau
    for tt in np.linspace(0, 3 * tau, 31):
        assert f(tau) <= f(tt) + 1e-12 * f0
    # g is Z^T r with the dense Z
    r = oracle.residual(x, d, z, dtype=np.float64)
    gd = sum(dense_Z(z[n], s).T @ r[n].ravel() for n in range(N))
    assert rel_err(g.ravel(), gd) < 1e-12
    assert abs(zg2 - sum(np.sum((dense_Z(z[n], s) @ g.ravel()) ** 2) for n in range(N))) < 1e-10 * zg2
    # projection onto the unit ball per filter
    e = d - tau * g
    nrm = np.sqrt((e * e).sum(axis=(1, 2), keepdims=True))
    assert rel_err(d_new, e / np.maximum(1.0, nrm)) < 1e-14
    assert (np.sqrt((d_new ** 2).sum(axis=(1, 2))) <= 1 + 1e-12).all()


def test_filter_step_zero_codes_leave_filters():
    x, d, z = random_problem(61, 2, 3, 3, 6, 6, dtype=np.float32)
    d_new, tau, g, _ = oracle.filter_step(x, d, np.zeros_like(z), 0.0, dtype=np.float32)
    assert not g.any() and tau == 0.0
    assert np.array_equal(d_new, d)


def test_filter_step_inside_ball_unchanged_by_projection():
    x, d, z = random_problem(62, 1, 2, 3, 6, 6, dtype=np.float64)
    d = d * 0.5  # strictly inside the ball
    step = 1e-6
    d_new, tau, g, _ = oracle.filter_step(x, d, z, step, dtype=np.float64)
    assert rel_err(d_new, d - tau * g) < 1e-15


def test_filter_step_fp32_projection_bound():
    cfg = CONFIGS["tiny"]
    x = make_images(cfg)
    d = make_filters(cfg)
    z = np.random.default_rng(3).standard_normal(make_codes(cfg).shape).astype(np.float32)
    d_new, _, _, _ = oracle.filter_step(x, d, z, 0.0, dtype=np.float32)
    assert (np.sqrt((d_new.astype(np.float64) ** 2).sum(axis=(1, 2))) <= 1 + 1e-6).all()


def test_tiny_iteration_objective_monotone():
    """Alternating masked ISTA (tau = 1/L_hat) + line-searched projected filter step on the
    tiny config: F(z^t, d^t) non-increasing over 15 iterations at p = 1 and p = 0.5
    (SPEC acceptance #5 adapted to 1/L steps)."""
    cfg = CONFIGS["tiny"]
    x = make_images(cfg)
    for p in (1.0, 0.5):
        d = make_filters(cfg)
        z = make_codes(cfg)
        F_prev = oracle.objective(x, d, z, cfg.lam)[0]
        for t in range(1, 16):
            it = oracle.iteration(x, d, z, cfg.lam, p, mask_seed(cfg), t)
            z, d = it["z"], it["d"]
            F = it["F"][0]
            assert F <= F_prev * (1 + 1e-6)
            F_prev = F

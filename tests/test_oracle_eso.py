"""Pins of the oracle's ESO step rule (reading E1):
tau_k = 1 / (p L_D + (1-p) ||d_k||^2) for the codes of filter k, the parallel-coordinate-descent
step for independent Bernoulli(p) sampling (the mini-batch coordinate descent the paper cites,
P:620-623).  Independent of the oracle:
  * p = 1 reduces to the Lipschitz step of reading R8 (bit for bit);
  * the ESO inequality behind the rule holds for Bernoulli sampling, by exact enumeration of all
    subsets on a dense sub-matrix, the expectation equals its closed form, and dropping the p L
    term breaks the bound;
  * the expected objective does not increase (Monte-Carlo over masks), while the step that drops
    the (1-p)||d_k||^2 term does increase it;
  * as p -> 0 the step of an isolated interior code is the exact 1-D minimiser of F along that
    coordinate, found by a bracketing search on the dense matrix.
"""
import itertools

import numpy as np
import pytest

import oracle
from synth import random_problem
from tests._dense import dense_D


def test_eso_equals_lipschitz_step_at_p1():
    x, d, z = random_problem(11, 2, 4, 5, 14, 13, code_density=0.3)
    z1, t1 = oracle.code_step(x, d, z, 0.2, 0.0, 1.0, 9, 4)
    z2, tk = oracle.code_step(x, d, z, 0.2, 0.0, 1.0, 9, 4, rule="eso")
    assert np.all(tk == t1)
    assert np.array_equal(z1, z2)


@pytest.mark.parametrize("p", [0.1, 0.5])
def test_eso_inequality_bernoulli_enumeration(p):
    """E ||A h_[S]||^2 <= p sum_i (p L + (1-p) ||A_i||^2) h_i^2 over all 2^n subsets S."""
    rng = np.random.default_rng(3)
    _, d, _ = random_problem(5, 1, 2, 3, 4, 4)
    A = dense_D(d.astype(np.float64), 4, 4)[:, rng.choice(2 * 36, 12, replace=False)]
    n = A.shape[1]
    L = np.linalg.norm(A, 2) ** 2
    cn = (A ** 2).sum(axis=0)
    for trial in range(5):
        h = rng.standard_normal(n)
        e = 0.0
        for S in itertools.product([0, 1], repeat=n):
            S = np.array(S, dtype=bool)
            pr = p ** S.sum() * (1 - p) ** (n - S.sum())
            e += pr * np.sum((A[:, S] @ h[S]) ** 2)
        bound = p * np.sum((p * L + (1 - p) * cn) * h ** 2)
        assert e <= bound * (1 + 1e-12)
        # the closed form of the expectation (no bound)
        exact = p * p * np.sum((A @ h) ** 2) + p * (1 - p) * np.sum(cn * h ** 2)
        assert abs(e - exact) <= 1e-10 * exact
    # along the top singular direction the bound needs its p L term
    if p < 0.5:
        w, V = np.linalg.eigh(A.T @ A)
        h = V[:, -1]
        exact = p * p * np.sum((A @ h) ** 2) + p * (1 - p) * np.sum(cn * h ** 2)
        swapped = p * np.sum(((1 - p) * cn + p * L) * h ** 2)
        assert exact <= swapped * (1 + 1e-12)  # still an upper bound here ...
        wrong = p * np.sum((p * cn + (1 - p) * 0.0) * h ** 2)  # ... but dropping L is not
        assert exact > wrong


def _F(x, d, z, lam):
    return oracle.objective(x, d, z, lam, dtype=np.float64)[0]


def test_eso_expected_decrease_and_dropped_term_increase():
    """From z = 0 the ESO step decreases F on average over masks; tau = 1/(p L) (the (1-p)||d_k||^2
    term dropped) overshoots every selected coordinate by more than 2x and increases it."""
    x, d, z = random_problem(21, 1, 3, 5, 12, 12, code_density=0.0)
    x = x.astype(np.float64); d = d.astype(np.float64); z = z.astype(np.float64)
    lam, p = 0.01, 0.05
    F0 = _F(x, d, z, lam)
    Fs = [_F(x, d, oracle.code_step(x, d, z, lam, 0.0, p, 77, t, dtype=np.float64, rule="eso")[0], lam)
          for t in range(400)]
    assert np.mean(Fs) < F0
    L = oracle.lipschitz(d)
    assert 1.0 / (p * L) > 2.0  # every coordinate (curvature ||d_k||^2 = 1) overshoots
    Fw = [_F(x, d, oracle.code_step(x, d, z, lam, 1.0 / (p * L), p, 77, t, dtype=np.float64)[0], lam)
          for t in range(400)]
    assert np.mean(Fw) > F0


def test_eso_small_p_is_exact_coordinate_minimiser():
    K, s, H, W = 2, 3, 40, 40
    x, d, z = random_problem(31, 1, K, s, H, W, code_density=0.2)
    x = x.astype(np.float64); d = d.astype(np.float64); z = z.astype(np.float64)
    lam, p = 0.05, 1e-3
    A = dense_D(d, H, W)
    Hc, Wc = H + s - 1, W + s - 1
    P = s - 1
    chosen = None
    for t in range(200):
        m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 5, t), K, Hc, Wc).ravel()
        if 2 <= m.sum() <= 8:
            chosen = (t, m)
            break
    assert chosen is not None
    t, m = chosen
    zo, tk = oracle.code_step(x, d, z, lam, 0.0, p, 5, t, dtype=np.float64, rule="eso")
    sel = np.flatnonzero(m)
    zf = z.ravel()
    b = x.ravel()
    checked = 0
    for i in sel:
        k, rem = divmod(i, Hc * Wc)
        u, v = divmod(rem, Wc)
        if not (P <= u < H and P <= v < W):
            continue  # border code: its column norm is below ||d_k||^2
        others = [j for j in sel if j != i]
        if others and np.abs(A[:, others].T @ A[:, i]).max() > 0:
            continue  # footprint overlaps another selected code
        # exact 1-D minimiser of F along coordinate i (others fixed) by bracketing on the dense matrix
        ri = A @ zf - b - A[:, i] * zf[i]

        def f1(w):
            return 0.5 * np.sum((ri + A[:, i] * w) ** 2) + lam * abs(w)
        lo, hi = zf[i] - 50.0, zf[i] + 50.0
        for _ in range(200):  # ternary search on a convex function
            a1, a2 = lo + (hi - lo) / 3, hi - (hi - lo) / 3
            if f1(a1) <= f1(a2):
                hi = a2
            else:
                lo = a1
        wstar = 0.5 * (lo + hi)
        if abs(wstar) < 1e-9:
            wstar = 0.0
        # tau_k differs from 1/||d_k||^2 by p L / ||d_k||^2 relative; the step is exact up to that
        rel = p * oracle.lipschitz(d) / np.sum(d[k] ** 2)
        assert abs(zo.ravel()[i] - wstar) <= 2 * rel * max(1.0, abs(wstar - zf[i])) + 1e-9
        checked += 1
    assert checked >= 1


def test_sector8_code_step_is_masked_ista_on_the_sector_mask():
    """NEXT-4 (ii): the code step under block-structured masks is the textbook ISTA update on the
    coordinates the sector mask selects (dense matrix), the other codes untouched."""
    K, s, H, W = 2, 3, 10, 9
    x, d, z = random_problem(41, 1, K, s, H, W, code_density=0.3)
    x = x.astype(np.float64); d = d.astype(np.float64); z = z.astype(np.float64)
    lam, p, seed, t = 0.1, 0.3, 9, 2
    zo, tau = oracle.code_step(x, d, z, lam, 0.0, p, seed, t, dtype=np.float64, mask="sector8")
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, t, mode="sector8"), K, Hc, Wc).ravel()
    assert m.any() and (~m).any()
    A = dense_D(d, H, W)
    zf = z.ravel()
    w = zf - tau * (A.T @ (A @ zf - x.ravel()))
    ista = np.sign(w) * np.maximum(np.abs(w) - tau * lam, 0.0)
    expect = np.where(m, ista, zf)
    assert np.allclose(zo.ravel(), expect, rtol=0, atol=1e-12 * max(1.0, np.abs(expect).max()))

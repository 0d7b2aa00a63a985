"""Pins of the oracle's online surrogates (Eq.7) and the surrogate filter update (Eq.8)
(PAPER.md P:366-389), independent of the oracle:
  * t = 1 from an empty state: C = Z^T Z and B = Z^T x of the dense Z matrix (tests/_dense.py);
  * after three mini-batches C and B equal the direct averages (1/t) sum_i Z_i^T Z_i, Z_i^T x_i;
  * the Eq.8 objective 1/2 d^T C d - d^T B equals (1/t) sum_i 1/2||x_i - Z_i d||^2 - (1/t) sum_i
    1/2||x_i||^2 (the full-history objective up to its constant);
  * with C = I the surrogate update returns B projected filter by filter on the unit ball;
  * at t = 1 the surrogate sweep reproduces the batch block-coordinate sweep (pinned separately).
"""
import numpy as np

import oracle
from synth import random_problem
from tests._dense import dense_Z


def _blocked(Zt_Z, K, M):
    """(KM x KM) row-major with index k*M + t -> block-major [K][K][M][M]."""
    return Zt_Z.reshape(K, M, K, M).transpose(0, 2, 1, 3)


def _batch(seed, N=2, K=3, s=3, H=7, W=6):
    return random_problem(seed, N, K, s, H, W, code_density=0.4)


def _dense_all(x, z, s):
    Z = np.concatenate([dense_Z(z[n], s) for n in range(z.shape[0])], axis=0)
    return Z, x.reshape(-1).astype(np.float64)


def test_first_update_is_the_batch_gram():
    x, d, z = _batch(1)
    K, M = 3, 9
    C = np.zeros((K, K, M, M)); B = np.zeros((K, M))
    oracle.surrogate_update(x, z, C, B, 1, dtype=np.float64)
    Z, xv = _dense_all(x, z, 3)
    assert np.allclose(C, _blocked(Z.T @ Z, K, M), rtol=1e-12, atol=1e-12)
    assert np.allclose(B.ravel(), Z.T @ xv, rtol=1e-12, atol=1e-12)


def test_three_updates_are_the_running_average_and_the_objective_matches():
    K, M = 3, 9
    C = np.zeros((K, K, M, M)); B = np.zeros((K, M))
    Cs, Bs, batches = 0, 0, []
    for t in range(1, 4):
        x, d, z = _batch(10 + t)
        oracle.surrogate_update(x, z, C, B, t, dtype=np.float64)
        Z, xv = _dense_all(x, z, 3)
        Cs = Cs + Z.T @ Z; Bs = Bs + Z.T @ xv
        batches.append((Z, xv))
    assert np.allclose(C, _blocked(Cs / 3, K, M), rtol=1e-12, atol=1e-12)
    assert np.allclose(B.ravel(), Bs / 3, rtol=1e-12, atol=1e-12)
    dv = np.random.default_rng(3).standard_normal(K * M)
    Cf = C.transpose(0, 2, 1, 3).reshape(K * M, K * M)
    sur = 0.5 * dv @ Cf @ dv - dv @ B.ravel()
    full = np.mean([0.5 * np.sum((xv - Z @ dv) ** 2) - 0.5 * np.sum(xv ** 2) for Z, xv in batches])
    assert abs(sur - full) <= 1e-10 * max(1.0, abs(full))


def test_identity_surrogate_returns_projected_b():
    K, s = 4, 3
    M = s * s
    C = np.zeros((K, K, M, M))
    for k in range(K):
        C[k, k] = np.eye(M)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((K, M)) * np.array([0.1, 0.2, 2.0, 5.0])[:, None]
    d0 = rng.standard_normal((K, s, s))
    dn, flags = oracle.filter_step_surrogate(C, B, d0, dtype=np.float64)
    expect = B / np.maximum(1.0, np.linalg.norm(B, axis=1))[:, None]
    assert not flags.any()
    assert np.allclose(dn.reshape(K, M), expect, rtol=0, atol=1e-8)


def test_first_surrogate_sweep_equals_the_batch_sweep():
    x, d, z = _batch(7)
    K, M = 3, 9
    C = np.zeros((K, K, M, M)); B = np.zeros((K, M))
    oracle.surrogate_update(x, z, C, B, 1, dtype=np.float64)
    d1, _ = oracle.filter_step_surrogate(C, B, d, dtype=np.float64)
    d2, _ = oracle.filter_step_bcd(x, d, z, dtype=np.float64)
    assert np.abs(d1 - d2).max() <= 1e-9

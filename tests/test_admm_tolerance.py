"""Derivation of the ADMM parity tolerance (reading A7), on the CPU.

One ADMM code step (10 iterations, 5 CG steps, rho = 10 lambda, alpha = 1.8) applies
(A^T A + rho I) 50 times.  Here it runs in fp64 on the dense matrix of tests/_dense.py, once
exactly and once with a relative perturbation eps on every A v and A^T e (the model of a GPU dense
pass's rounding), and the relative change of the output is measured.  The amplification stays
near 10, so a per-application error of ~1e-6 -- what the fp16 / tf32 3-term splits with fp32
accumulation give after cancellation -- maps to ~1e-5 in the codes; tests/test_gpu_admm.py uses
2e-5.  The test pins the amplification range the tolerance rests on.
"""
import numpy as np
import pytest

from synth import random_problem
from tests._dense import dense_D, soft


def _admm(A, b, w0, lam, rho, alpha, na, nc, eps, rng):
    def op(v):
        e = A @ v
        if eps:
            e = e * (1 + eps * rng.standard_normal(e.shape))
        g = A.T @ e
        if eps:
            g = g * (1 + eps * rng.standard_normal(g.shape))
        return g + rho * v
    atb = A.T @ b
    w = w0.copy(); y = w0.copy(); u = np.zeros_like(w)
    for _ in range(na):
        r = atb + rho * (y - u) - op(w)
        pv = r.copy(); rr = r @ r
        for _ in range(nc):
            if rr <= 0:
                break
            q = op(pv)
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
    return y


@pytest.mark.parametrize("shape", [(8, 5, 32, 32), (12, 7, 24, 24)])
def test_admm_error_amplification(shape):
    K, s, H, W = shape
    x, d, z = random_problem(300 + K, 1, K, s, H, W, code_density=0.3)
    A = dense_D(d.astype(np.float64), H, W)
    b = x[0].ravel().astype(np.float64)
    w0 = z[0].ravel().astype(np.float64)
    lam = 0.2
    y0 = _admm(A, b, w0, lam, 10 * lam, 1.8, 10, 5, 0.0, None)
    eps = 1e-6
    amp = max(np.linalg.norm(_admm(A, b, w0, lam, 10 * lam, 1.8, 10, 5, eps, np.random.default_rng(i)) - y0)
              / np.linalg.norm(y0) / eps for i in range(3))
    assert 2.0 < amp < 20.0, amp

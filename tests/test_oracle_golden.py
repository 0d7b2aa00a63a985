"""The oracle reproduces the hand-derived worked example in tests/golden/ (fp64 build)."""
import json
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_worked_example.json")


def _load():
    g = json.load(open(GOLDEN))
    d = np.array(g["d"], dtype=np.float64)
    z = np.zeros((1, 1, 4, 4))
    for u, v, val in g["z_nonzeros"]:
        z[0, 0, u, v] = val
    x = np.array(g["x"], dtype=np.float64)[None]
    return g, d, z, x


def test_golden_residual_objective_gradients():
    g, d, z, x = _load()
    assert np.array_equal(oracle.residual(None, d, z, dtype=np.float64)[0], np.array(g["Dz"], dtype=float))
    r = oracle.residual(x, d, z, dtype=np.float64)
    assert np.array_equal(r[0], np.array(g["r"], dtype=float))
    F, fit, l1 = oracle.objective(x, d, z, g["lam"], dtype=np.float64)
    assert (F, fit, l1) == (g["F"], g["half_r2"], g["lam"] * g["l1"])
    dt = oracle.dtr(d, r, dtype=np.float64)
    for u, v, val in g["dtr_at"]:
        assert dt[0, 0, u, v] == val
    gr = oracle.filter_grad(r, z, dtype=np.float64)
    assert np.array_equal(gr[0], np.array(g["g"], dtype=float))


def test_golden_code_step():
    g, d, z, x = _load()
    z1, tau = oracle.code_step(x, d, z, g["lam"], g["tau"], 1.0, 0, 1, dtype=np.float64)
    for u, v, val in g["z_after_code_step_p1"]:
        assert abs(z1[0, 0, u, v] - val) < 1e-15

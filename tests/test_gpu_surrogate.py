"""GPU parity of the online surrogates (Eq.7) and the Eq.8 filter update (
include/csc.h csc_surrogate_*) against the oracle (pinned in
tests/test_oracle_surrogate.py).

Bar: C and B are fp64 sums of exact products on both sides (only the summation order differs):
1e-12 relative; filters after the Eq.8 sweeps within 1e-5 relative (R9); flags equal.
"""
import numpy as np
import pytest

import oracle
from synth import random_problem
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    from paper_1909_00145_b200 import build as b
    b.build()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def _t(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("gram", ["lag", "direct"])
@pytest.mark.parametrize("shape", [(2, 5, 5, 20, 24), (3, 3, 3, 10, 12), (1, 8, 7, 16, 16), (2, 4, 11, 12, 12)])
def test_surrogate_update_and_filter_step_parity(torch_dev, shape, gram, monkeypatch):
    import torch
    import paper_1909_00145_b200 as pkg
    if gram == "direct":
        monkeypatch.setenv("CSC_BCD_GRAM", "direct")
    N, K, s, H, W = shape
    M = s * s
    ctx = pkg.Context(N, K, s, H, W, device=0)
    ctx.surrogate_reset()
    C = np.zeros((K, K, M, M)); B = np.zeros((K, M))
    d = None
    for t in range(1, 4):
        x, d0, z = random_problem(600 + 10 * t + K, N, K, s, H, W, code_density=0.3)
        if d is None:
            d = d0
        if t == 2 and K > 2:
            z[:, 2] = 0.0
        ctx.surrogate_update(_t(x, torch_dev), _t(z, torch_dev))
        oracle.surrogate_update(x, z, C, B, t)
    Cg = torch.zeros(K * K * M * M, dtype=torch.float64, device=torch_dev)
    Bg = torch.zeros(K * M, dtype=torch.float64, device=torch_dev)
    tg = ctx.read_surrogate(Cg, Bg)
    torch.cuda.synchronize()
    assert tg == 3
    assert np.abs(Cg.cpu().numpy() - C.ravel()).max() <= 1e-12 * np.abs(C).max()
    assert np.abs(Bg.cpu().numpy() - B.ravel()).max() <= 1e-12 * np.abs(B).max()
    dt = _t(d, torch_dev)
    flags = ctx.filter_step_surrogate(dt, sweeps=2, want_flags=True)
    do, fo = oracle.filter_step_surrogate(C, B, d, sweeps=2)
    torch.cuda.synchronize()
    err = rel_err(dt.cpu().numpy(), do)
    print(f"surrogate {shape}: d rel err {err:.3e}")
    assert err < 1e-5, err
    assert list(flags) == list(fo)
    ctx.close()


def test_surrogate_errors(torch_dev):
    import paper_1909_00145_b200 as pkg
    x, d, z = random_problem(2, 1, 2, 3, 8, 8)
    ctx = pkg.Context(1, 2, 3, 8, 8, device=0)
    with pytest.raises(pkg.CSCError):
        ctx.filter_step_surrogate(_t(d, torch_dev))  # no update yet
    ctx.surrogate_update(_t(x, torch_dev), _t(z, torch_dev))
    with pytest.raises(pkg.CSCError):
        ctx.filter_step_surrogate(_t(d, torch_dev), sweeps=0)
    ctx.close()

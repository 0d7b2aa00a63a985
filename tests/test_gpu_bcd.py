"""GPU parity of the projected block-coordinate filter update (include/csc.h
csc_filter_step_bcd) against oracle.filter_step_bcd (pinned in tests/test_oracle_bcd.py).

Bar: filters within 1e-5 relative (norm-wise, R9) after one and after three sweeps; flags equal;
the following objective (through the hot path's dense pass) within 1e-5 of the oracle's.
"""
import numpy as np
import pytest

import oracle
from synth import random_problem
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-5


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
@pytest.mark.parametrize("sweeps", [1, 3])
@pytest.mark.parametrize("shape", [(3, 5, 5, 70, 130), (2, 17, 11, 40, 44), (4, 8, 5, 32, 32), (1, 9, 3, 33, 47),
                                   (2, 4, 11, 11, 11), (1, 3, 1, 9, 12)])
def test_bcd_filter_step_parity(torch_dev, shape, sweeps, gram, monkeypatch):
    """gram: the lag-structured Gram (default where H, W > P) or the direct per-tap-pair sum."""
    import torch
    import paper_1909_00145_b200 as pkg
    if gram == "direct":
        monkeypatch.setenv("CSC_BCD_GRAM", "direct")
    N, K, s, H, W = shape
    x, d, z = random_problem(500 + K, N, K, s, H, W, code_density=0.3)
    if K > 2:
        z[:, 1] = 0.0  # a filter without codes: left unchanged and flagged
    ctx = pkg.Context(N, K, s, H, W, device=0)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    flags = ctx.filter_step_bcd(xt, dt, zt, sweeps=sweeps, want_flags=True)
    dn, fo = oracle.filter_step_bcd(x, d, z, sweeps=sweeps)
    torch.cuda.synchronize()
    err = rel_err(dt.cpu().numpy(), dn)
    print(f"bcd {shape} sweeps={sweeps} {gram}: rel err {err:.3e}")
    assert err < TOL, err
    assert list(flags) == list(fo)
    F = ctx.objective(xt, dt, zt, 0.3)
    Fo = oracle.objective(x, dn, z, 0.3)
    assert abs(F[0] - Fo[0]) <= TOL * abs(Fo[0])
    ctx.close()


def test_bcd_argument_errors(torch_dev):
    import paper_1909_00145_b200 as pkg
    x, d, z = random_problem(1, 1, 2, 3, 8, 8)
    ctx = pkg.Context(1, 2, 3, 8, 8, device=0)
    with pytest.raises(pkg.CSCError):
        ctx.filter_step_bcd(_t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev), sweeps=0)
    ctx.close()


def test_next_rows_with_an_empty_local_batch(torch_dev):
    """n_local = 0 (a rank with no images): the ADMM step is a no-op, the BCD sweep leaves every
    filter unchanged and flagged (no codes), and a surrogate update with no images keeps C = 0."""
    import torch
    import paper_1909_00145_b200 as pkg
    from synth import CONFIGS, make_filters
    K, s = 4, 3
    ctx = pkg.Context(0, K, s, 8, 8, device=0)
    d = _t(make_filters(CONFIGS["tiny"].with_(K=K, s=s)), torch_dev)
    d0 = d.clone()
    e = torch.zeros(0, device=torch_dev)
    ctx.code_step_admm(e, d, e, 0.5, 0.5, 1, 1)
    flags = ctx.filter_step_bcd(e, d, e, want_flags=True)
    assert flags == [1] * K
    ctx.surrogate_update(e, e)
    C = torch.ones(K * K * s ** 4, dtype=torch.float64, device=torch_dev)
    B = torch.ones(K * s * s, dtype=torch.float64, device=torch_dev)
    assert ctx.read_surrogate(C, B) == 1
    torch.cuda.synchronize()
    assert torch.equal(d, d0)
    assert float(C.abs().max()) == 0.0 and float(B.abs().max()) == 0.0
    ctx.close()

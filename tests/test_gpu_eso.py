"""GPU parity of the ESO step rule (include/csc.h csc_set_step_rule;
DESIGN.md reading E1) against the oracle (pinned in tests/test_oracle_eso.py).

Bar: as the hot path's code step (BASELINE.json north_star): codes within 1e-5 relative
(norm-wise, R9), unselected codes bit-identical (R2), the per-filter step sizes within 1e-6
relative (they are fp32 roundings of the same fp64 expression, with L_D from the same DFT grid
evaluated in a different summation order), and a 20-iteration trajectory with the ESO rule.
"""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed, random_problem
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


@pytest.mark.parametrize("path", ["half", "tc", "simt"])
@pytest.mark.parametrize("shape,p", [((3, 5, 5, 70, 130), 0.1), ((2, 17, 11, 100, 100), 0.2),
                                     ((1, 9, 3, 33, 47), 0.5), ((2, 130, 7, 20, 300), 0.05),
                                     ((1, 100, 11, 40, 11), 0.3), ((4, 8, 5, 32, 32), 1.0)])
def test_eso_code_step_parity(torch_dev, shape, p, path, monkeypatch):
    import torch
    import paper_1909_00145_b200 as pkg
    monkeypatch.setenv("CSC_CODE_PATH", path)
    N, K, s, H, W = shape
    x, d, z = random_problem(400 + K, N, K, s, H, W, code_density=0.3)
    seed, it, lam = 4242, 7, 0.2
    ctx = pkg.Context(N, K, s, H, W, device=0)
    ctx.set_step_rule("eso")
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    tau0 = ctx.code_step(xt, dt, zt, lam, p, seed, it, want_step=True)
    tk = torch.zeros(K, dtype=torch.float32, device=torch_dev)
    ctx.read_step_z(tk)
    torch.cuda.synchronize()
    zo, tko = oracle.code_step(x, d, z, lam, 0.0, p, seed, it, rule="eso")
    assert np.abs(tk.cpu().numpy() - tko).max() <= 1e-6 * tko.max()
    assert abs(tau0 - tko[0]) <= 1e-6 * tko[0]
    zg = zt.cpu().numpy()
    assert rel_err(zg, zo) < TOL
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, it), K, Hc, Wc)
    for n in range(N):
        assert np.array_equal(zg[n][~m], z[n][~m])
    # back to the Lipschitz rule: the same call reproduces the R8 step
    ctx.set_step_rule("lipschitz")
    zt2 = _t(z, torch_dev)
    ctx.invalidate()
    ctx.code_step(xt, dt, zt2, lam, p, seed, it)
    zo2, _ = oracle.code_step(x, d, z, lam, 0.0, p, seed, it)
    torch.cuda.synchronize()
    assert rel_err(zt2.cpu().numpy(), zo2) < TOL
    ctx.close()


def test_eso_trajectory_20_iterations(torch_dev):
    """Config 1 shape at p = 0.2: 20 iterations of ESO code step + filter step, every one compared
    with the oracle's code_step(rule="eso") + filter_step + objective."""
    import torch
    import paper_1909_00145_b200 as pkg
    cfg = CONFIGS["tiny"]
    p = 0.2
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
    ctx.set_step_rule("eso")
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    for t in range(1, 21):
        F, _ = ctx.iterate(xt, dt, zt, cfg.lam, p, seed, t)
        z, _ = oracle.code_step(x, d, z, cfg.lam, 0.0, p, seed, t, rule="eso")
        d, _, _, _ = oracle.filter_step(x, d, z)
        Fo = oracle.objective(x, d, z, cfg.lam)
        torch.cuda.synchronize()
        assert rel_err(zt.cpu().numpy(), z) < TOL, t
        assert rel_err(dt.cpu().numpy(), d) < TOL, t
        assert abs(F[0] - Fo[0]) <= TOL * abs(Fo[0]), t
    ctx.close()


def test_step_rule_argument_error(torch_dev):
    import paper_1909_00145_b200 as pkg
    ctx = pkg.Context(1, 2, 3, 8, 8, device=0)
    with pytest.raises(pkg.CSCError):
        ctx._check(ctx._L.csc_set_step_rule(ctx._h, 7))
    ctx.close()


# ---- NEXT-4 (ii): block-structured masks (a labelled deviation, E5)
@pytest.mark.parametrize("K,Hc,Wc", [(8, 36, 36), (3, 7, 9), (5, 41, 67), (100, 110, 110)])
@pytest.mark.parametrize("p", [0.1, 0.5, 1.0])
def test_sector8_mask_bits_bit_exact(torch_dev, K, Hc, Wc, p):
    import torch
    import paper_1909_00145_b200 as pkg
    s = 3
    ctx = pkg.Context(1, K, s, Hc - s + 1, Wc - s + 1, device=0)
    ctx.set_mask_mode("sector8")
    out = torch.zeros((K * Hc * Wc + 31) // 32, dtype=torch.int32, device=torch_dev)
    for seed, it in [(0, 0), (0x0123456789ABCDEF, 7)]:
        ctx.mask_bits(it, p, seed, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle.mask_bits(K, Hc, Wc, p, seed, it, "sector8"))
    ctx.close()


@pytest.mark.parametrize("path", ["half", "tc", "simt"])
@pytest.mark.parametrize("shape,p", [((3, 5, 5, 70, 130), 0.1), ((2, 17, 11, 100, 100), 0.2),
                                     ((1, 9, 3, 33, 47), 0.5), ((2, 130, 7, 20, 300), 0.1)])
def test_sector8_code_step_parity(torch_dev, shape, p, path, monkeypatch):
    import torch
    import paper_1909_00145_b200 as pkg
    monkeypatch.setenv("CSC_CODE_PATH", path)
    N, K, s, H, W = shape
    x, d, z = random_problem(700 + K, N, K, s, H, W, code_density=0.3)
    seed, it, lam = 31337, 4, 0.2
    ctx = pkg.Context(N, K, s, H, W, device=0)
    ctx.set_mask_mode("sector8")
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    ctx.code_step(xt, dt, zt, lam, p, seed, it)
    zo, _ = oracle.code_step(x, d, z, lam, 0.0, p, seed, it, mask="sector8")
    torch.cuda.synchronize()
    zg = zt.cpu().numpy()
    assert rel_err(zg, zo) < TOL
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, it, "sector8"), K, Hc, Wc)
    for n in range(N):
        assert np.array_equal(zg[n][~m], z[n][~m])
    with pytest.raises(pkg.CSCError):
        ctx.code_step_admm(xt, dt, zt, lam, p, seed, it)  # ADMM keeps the per-entry masks of Eq.2
    ctx.close()


def test_eso_with_sector_masks_rejected(torch_dev):
    """The ESO step (E1) holds for independent per-code sampling only: with sector masks the
    code step refuses it (CSC_ERR_ARG, no side effects); an explicit step is still accepted."""
    import torch
    import paper_1909_00145_b200 as pkg
    x, d, z = random_problem(5, 1, 6, 5, 20, 24, code_density=0.3)
    ctx = pkg.Context(1, 6, 5, 20, 24, device=0)
    ctx.set_step_rule("eso")
    ctx.set_mask_mode("sector8")
    xt, dt, zt = (torch.from_numpy(np.ascontiguousarray(a)).to(torch_dev) for a in (x, d, z))
    z0 = zt.clone()
    with pytest.raises(pkg.CSCError) as ei:
        ctx.code_step(xt, dt, zt, 0.2, 0.5, 1, 1)
    assert ei.value.status == 1
    torch.cuda.synchronize()
    assert torch.equal(zt, z0)
    ctx.code_step(xt, dt, zt, 0.2, 0.5, 1, 1, step_z=0.01)
    ctx.close()

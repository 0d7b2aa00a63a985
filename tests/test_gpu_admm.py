"""GPU parity of the ADMM masked-LASSO code solver (
include/csc.h csc_code_step_admm) against oracle.admm_code_step (pinned in tests/test_oracle_admm.py).

Bar: codes within TOL_ADMM = 1e-5 relative (norm-wise, reading R9) of the fp64 oracle after one step
of 10 ADMM x 5 CG iterations (the north_star bar); codes off the mask bit-identical (R2).  One step
applies the operator 50 times and amplifies a per-application relative error ~7-10x
(tests/test_admm_tolerance.py, reading A7); the operator's tensor-core passes therefore
accumulate the hi*hi products and the cross products of the fp16 split in separate TMEM
accumulators (reading T3), which keeps the per-application error near 1e-7.
"""
import numpy as np
import pytest

import oracle
from synth import random_problem
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TOL_ADMM = 1e-5


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


SHAPES = [((3, 5, 5, 70, 130), 0.1), ((2, 17, 11, 100, 100), 0.2), ((4, 8, 5, 32, 32), 1.0),
          ((1, 9, 3, 33, 47), 0.5), ((2, 4, 11, 11, 11), 0.05), ((2, 130, 7, 20, 300), 0.1),
          ((1, 100, 11, 40, 11), 0.3), ((2, 16, 7, 64, 64), 1.0), ((1, 32, 11, 50, 50), 1.0),
          ((3, 24, 9, 40, 72), 0.5)]


@pytest.mark.parametrize("shape,p", [((2, 17, 11, 100, 100), 0.2), ((1, 9, 3, 33, 47), 0.5),
                                     ((2, 16, 7, 64, 64), 1.0)])
@pytest.mark.parametrize("var,modes", [("CSC_ADMM_EXPAND", ["float4", "scalar"])])
def test_admm_data_movement_bit_identical(torch_dev, shape, p, var, modes, monkeypatch):
    """Variants that only move the same values differently give identical z: the staged float4
    expansion vs the scalar one."""
    import torch
    import paper_1909_00145_b200 as pkg
    N, K, s, H, W = shape
    x, d, z = random_problem(900 + K, N, K, s, H, W, code_density=0.3)
    out = []
    for mode in modes:
        monkeypatch.setenv(var, mode)
        ctx = pkg.Context(N, K, s, H, W, device=0)
        zt = _t(z, torch_dev)
        ctx.code_step_admm(_t(x, torch_dev), _t(d, torch_dev), zt, 0.2, p, 99, 3)
        torch.cuda.synchronize()
        out.append(zt.cpu().numpy())
        ctx.close()
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("dense", ["half", "simt", "dtr_simt", "explicit"])
@pytest.mark.parametrize("shape,p", SHAPES)
def test_admm_code_step_parity(torch_dev, shape, p, dense, monkeypatch):
    """dense: the operator A v on the fp16-split tensor-core pass ("half") or the SIMT pass; A^T e
    on the tensor cores (code_h plain mode + gather) unless "dtr_simt" (SIMT masked correlation)."""
    import torch
    import paper_1909_00145_b200 as pkg
    if dense == "simt":
        monkeypatch.setenv("CSC_DENSE_PATH", "simt")
    if dense == "dtr_simt":
        monkeypatch.setenv("CSC_ADMM_DTR", "simt")
    if dense == "explicit":
        monkeypatch.setenv("CSC_ADMM_RESID", "explicit")
    N, K, s, H, W = shape
    x, d, z = random_problem(300 + K, N, K, s, H, W, code_density=0.3)
    seed, it, lam = 777, 5, 0.2
    ctx = pkg.Context(N, K, s, H, W, device=0)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    ctx.code_step_admm(xt, dt, zt, lam, p, seed, it)
    torch.cuda.synchronize()
    zg = zt.cpu().numpy()
    zo = oracle.admm_code_step(x, d, z, lam, p, seed, it, dtype=np.float64)
    err = rel_err(zg, zo)
    print(f"admm {shape} p={p} {dense}: rel err {err:.3e}")
    assert err < TOL_ADMM, err
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, it), K, Hc, Wc)
    for n in range(N):
        assert np.array_equal(zg[n][~m], z[n][~m])
    ctx.close()


def test_admm_parameters_and_objective(torch_dev):
    """Explicit rho / alpha / iteration counts reach the oracle's result; a run followed by the
    hot path's objective matches the oracle's objective of the oracle's codes."""
    import torch
    import paper_1909_00145_b200 as pkg
    N, K, s, H, W = 2, 12, 7, 60, 52
    x, d, z = random_problem(41, N, K, s, H, W, code_density=0.2)
    ctx = pkg.Context(N, K, s, H, W, device=0)
    xt, dt = _t(x, torch_dev), _t(d, torch_dev)
    for rho, alpha, na, nc in [(0.5, 1.0, 3, 2), (4.0, 1.5, 7, 8), (0.0, 1.8, 1, 1)]:
        zt = _t(z, torch_dev)
        ctx.invalidate()
        ctx.code_step_admm(xt, dt, zt, 0.3, 0.4, 9, 2, rho=rho, alpha=alpha, n_admm=na, n_cg=nc)
        zo = oracle.admm_code_step(x, d, z, 0.3, 0.4, 9, 2, rho=(rho or None), alpha=alpha, n_admm=na, n_cg=nc,
                                   dtype=np.float64)
        torch.cuda.synchronize()
        err = rel_err(zt.cpu().numpy(), zo)
        print(f"admm rho={rho} alpha={alpha} {na}x{nc}: rel err {err:.3e}")
        assert err < TOL_ADMM, err
    F = ctx.objective(xt, dt, zt, 0.3)
    Fo = oracle.objective(x, d, zo, 0.3, dtype=np.float64)
    assert abs(F[0] - Fo[0]) <= TOL_ADMM * Fo[0]
    ctx.close()


def test_admm_argument_errors(torch_dev):
    import paper_1909_00145_b200 as pkg
    N, K, s, H, W = 1, 2, 3, 8, 8
    x, d, z = random_problem(1, N, K, s, H, W)
    ctx = pkg.Context(N, K, s, H, W, device=0)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    for kw in [dict(lam=0.0), dict(alpha=2.0), dict(alpha=0.0), dict(n_admm=0), dict(n_cg=0), dict(p=0.0),
               dict(rho=-1.0)]:
        args = dict(lam=0.1, p=0.5, alpha=1.8, n_admm=10, n_cg=5, rho=0.0)
        args.update(kw)
        with pytest.raises(pkg.CSCError):
            ctx.code_step_admm(xt, dt, zt, args["lam"], args["p"], 1, 1, rho=args["rho"], alpha=args["alpha"],
                               n_admm=args["n_admm"], n_cg=args["n_cg"])
    assert np.array_equal(zt.cpu().numpy(), z)
    ctx.close()


def test_admm_full_size_batch_config_image0(torch_dev):
    """BASELINE.json configs[1] at full size (10 images 100x100, K = 100, s = 11, p = 0.1): the ADMM
    step is per image (A2), so the oracle solves image 0 alone and its codes are compared with the
    GPU's image 0 from the full 10-image launch (the launch configuration bench.py uses)."""
    import torch
    import paper_1909_00145_b200 as pkg
    from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed
    cfg = CONFIGS["batch"]
    x, d = make_images(cfg), make_filters(cfg)
    rng = np.random.default_rng(5)
    z = make_codes(cfg)
    z[:] = (rng.standard_normal(z.shape) * (rng.random(z.shape) < 0.05)).astype(np.float32) * 0.1
    seed = mask_seed(cfg)
    ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    ctx.code_step_admm(xt, dt, zt, cfg.lam, cfg.p, seed, 3)
    torch.cuda.synchronize()
    zo = oracle.admm_code_step(x[:1], d, z[:1], cfg.lam, cfg.p, seed, 3, dtype=np.float64)
    err = rel_err(zt.cpu().numpy()[:1], zo)
    print(f"admm full-size batch image 0: rel err {err:.3e}")
    assert err < TOL_ADMM, err
    ctx.close()

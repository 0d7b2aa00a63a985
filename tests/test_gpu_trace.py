"""The per-iteration trace through the C ABI (paper_1909_00145_b200/trace.py; the Fig.1
caption's objective and time per iteration): every row's F, tau_z, tau_d match the
oracle's iteration (Alg.1) at the trajectory bars of tests/test_gpu_trajectories.py,
nnz equals the number of nonzero GPU codes, the phase times add up, and a traced run leaves the same
codes and filters as csc_iterate on a second context (same kernels, same order: bit-identical).
Also: csc_set_nvtx and csc_comm_check (world = 1) are accepted on a live context."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


def test_trace_matches_oracle_and_iterate():
    import torch
    import paper_1909_00145_b200 as pkg
    from paper_1909_00145_b200.trace import IterationTrace, run_traced
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["batch"].with_(K=24, N=3, H=40, W=36, p=0.3)
    x, d0, z0 = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    iters = 6
    ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
    ctx.set_nvtx(True)
    ctx.comm_check()
    xt, dt, zt = (torch.from_numpy(a).to(dev) for a in (x, d0, z0))
    tr = run_traced(ctx, xt, dt, zt, cfg.lam, cfg.p, seed, iters, start_iter=1)
    assert len(tr) == iters
    assert IterationTrace.read_csv(tr.to_csv()).rows == tr.rows
    # oracle iteration
    d, z = d0.copy(), z0.copy()
    for row in tr.rows:
        z, tau_z = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, seed, row["iter"])
        d, tau_d, _, _ = oracle.filter_step(x, d, z)
        F, fit, l1 = oracle.objective(x, d, z, cfg.lam)
        assert abs(row["F"] - F) <= 1e-5 * F, row
        assert abs(row["fit"] - fit) <= 1e-5 * fit, row
        assert abs(row["tau_z"] - tau_z) <= 1e-6 * tau_z, row
        assert abs(row["tau_d"] - tau_d) <= 1e-5 * tau_d, row
        assert row["ms_code"] > 0 and row["ms_filter"] > 0 and row["ms_obj"] > 0
        assert abs(row["ms_iter"] - (row["ms_code"] + row["ms_filter"] + row["ms_obj"])) <= 0.05 * row["ms_iter"] + 0.01
    assert tr.rows[-1]["nnz"] == int(torch.count_nonzero(zt).item())
    assert rel_err(zt.cpu().numpy(), z) < 1e-5
    assert rel_err(dt.cpu().numpy(), d) < 1e-5
    # the same iterations through csc_iterate on a second context: identical state
    c2 = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
    d2, z2 = torch.from_numpy(d0).to(dev), torch.from_numpy(z0).to(dev)
    for row in tr.rows:
        (F2, _, _), _ = c2.iterate(xt, d2, z2, cfg.lam, cfg.p, seed, row["iter"])
        assert F2 == row["F"]
    assert torch.equal(z2, zt) and torch.equal(d2, dt)
    ctx.set_nvtx(False)
    ctx.close()
    c2.close()


def test_count_nonzero_exact():
    import torch
    import paper_1909_00145_b200 as pkg
    torch.cuda.set_device(0)
    ctx = pkg.Context(1, 4, 3, 8, 8, device=0)
    g = torch.Generator().manual_seed(3)
    for n in (0, 1, 31, 4097, 1 << 20):
        v = torch.randn(n, generator=g) * (torch.rand(n, generator=g) < 0.3)
        v = v.to(torch.float32).cuda()
        assert ctx.count_nonzero(v) == int(torch.count_nonzero(v).item())
    ctx.close()

"""The image-sharded decomposition of the iteration on one GPU.

Codes are independent per image ("computing sparse codes is a data-independent process",
PAPER.md:661-663) and the mask is a counter-based function shared by every rank (reading R5), so a
world of n ranks computes exactly what one context over all images computes, provided the library
all-reduces three sums: the filter gradient g, ||Z g||^2 and the objective parts.  NCCL itself needs
several GPUs (and two ranks on one GPU may not wait on each other, B200_PROFILING.md); this test runs
the shard contexts side by side on one GPU with world = 1 and checks, through the C ABI, that the
per-shard partials the all-reduce would sum reproduce the single-context values:

  codes after the code step       shard codes == the full context's codes of those images
  g                               g_A + g_B == g_full
  ||Z g||^2 (global g)            zg2_A(g_full) + zg2_B(g_full) == zg2_full
  tau_d                           <g, g> / (zg2_A + zg2_B) == tau_d of the full context
  objective parts                 (fit, l1)_A + (fit, l1)_B == (fit, l1)_full
and that the shard split used by bench.py (paper_1909_00145_b200.dist.shard) covers the images.
"""
import numpy as np
import pytest

from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-6


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_1909_00145_b200 import build as b
    b.build()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


@pytest.mark.parametrize("K,s,H,W,N,world", [(24, 5, 40, 44, 5, 2), (100, 11, 60, 150, 7, 4), (12, 3, 33, 30, 3, 2)])
def test_sharded_partials_sum_to_full(dev, K, s, H, W, N, world):
    import torch
    import paper_1909_00145_b200 as pkg
    from paper_1909_00145_b200 import dist as cdist
    cfg = CONFIGS["batch"].with_(K=K, s=s, H=H, W=W, N=N, p=0.3)
    x = make_images(cfg)
    d0 = make_filters(cfg)
    seed = mask_seed(cfg)
    lam = cfg.lam

    def ctx(n):
        return pkg.Context(n, K, s, H, W, device=0)

    shards = [cdist.shard(N, world, r) for r in range(world)]
    assert shards[0][0] == 0 and shards[-1][1] == N and all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    full = ctx(N)
    parts = [ctx(b - a) for a, b in shards]
    xt = torch.from_numpy(x).to(dev)
    # two iterations' worth of codes so the codes are non-trivial
    zf = torch.from_numpy(make_codes(cfg)).to(dev)
    df = torch.from_numpy(d0).to(dev)
    zs = [torch.from_numpy(make_codes(cfg, b - a)).to(dev) for a, b in shards]
    ds = [torch.from_numpy(d0).to(dev) for _ in shards]
    xs = [xt[a:b].contiguous() for a, b in shards]
    for t in (1, 2):
        full.code_step(xt, df, zf, lam, cfg.p, seed, t)
        for c, xx, dd, zz in zip(parts, xs, ds, zs):
            c.code_step(xx, dd, zz, lam, cfg.p, seed, t)
        torch.cuda.synchronize()
        for (a, b), zz in zip(shards, zs):
            assert rel_err(zz.cpu().numpy(), zf[a:b].cpu().numpy()) < TOL, t
        if t == 1:
            # one filter step everywhere so that d moves the same way (the shard steps use their local g,
            # so re-sync the shard filters to the full context's after it)
            full.filter_step(xt, df, zf)
            for dd in ds:
                dd.copy_(df)
            for c in parts:
                c.invalidate()
    # the filter step of the full context, and the shard partials of the same step
    d_before = df.clone()
    tau_full = full.filter_step(xt, df, zf, want_step=True)
    g_full = torch.zeros(K * s * s, dtype=torch.float64, device=dev)
    full.read_grad(g_full)
    sc_full = full.read_scalars()
    g_sum = torch.zeros_like(g_full)
    zg2_sum = 0.0
    for c, xx, dd, zz in zip(parts, xs, ds, zs):
        c.filter_step(xx, dd, zz)  # local gradient (world = 1: no all-reduce)
        gl = torch.zeros_like(g_full)
        c.read_grad(gl)
        g_sum += gl
    assert rel_err(g_sum.cpu().numpy(), g_full.cpu().numpy()) < TOL
    for c, zz in zip(parts, zs):
        zg2_sum += c.zg_sumsq(zz, g_full)
    assert abs(zg2_sum - sc_full["zg2"]) <= TOL * sc_full["zg2"]
    gg = float((g_full * g_full).sum().item())
    assert abs(gg - sc_full["gg"]) <= 1e-12 * gg
    tau_sum = np.float32(gg / zg2_sum)
    assert abs(float(tau_sum) - tau_full) <= TOL * tau_full
    # the objective parts with the updated filters (the same on every rank)
    F_full = full.objective(xt, df, zf, lam)
    fit = l1 = 0.0
    for c, xx, zz in zip(parts, xs, zs):
        F = c.objective(xx, df, zz, lam)
        fit += F[1]
        l1 += F[2]
    assert abs(fit - F_full[1]) <= TOL * F_full[1]
    assert abs(l1 - F_full[2]) <= TOL * max(F_full[2], 1e-30)
    assert not torch.equal(d_before, df)
    for c in parts + [full]:
        c.close()

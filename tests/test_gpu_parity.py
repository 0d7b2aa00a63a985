"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star; SURVEY.md §8(c) "Required agreement"): masks bit-exact;
codes, filters and objective within 1e-5 relative (norm-wise, reading R9) per iteration;
the residual r and the gradient g within 1e-5; the step sizes tau_z, tau_d within 1e-6.
The 50-iteration trajectories of every BASELINE.json configuration are in
tests/test_gpu_trajectories.py.
"""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed, random_problem
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-5
TOL_TAU = 1e-6


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    from paper_1909_00145_b200 import build as b
    b.build()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def _ctx(N, K, s, H, W):
    import paper_1909_00145_b200 as pkg
    return pkg.Context(N, K, s, H, W, device=0)


def _t(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("K,Hc,Wc", [(8, 36, 36), (3, 7, 9), (5, 41, 67), (100, 110, 110), (2, 33, 29)])
@pytest.mark.parametrize("p", [0.05, 0.1, 0.5, 1.0])
def test_mask_bits_bit_exact(torch_dev, K, Hc, Wc, p):
    import torch
    s = 3
    ctx = _ctx(1, K, s, Hc - s + 1, Wc - s + 1)
    nwords = (K * Hc * Wc + 31) // 32
    out = torch.zeros(nwords, dtype=torch.int32, device=torch_dev)
    for seed, it in [(0, 0), (0x0123456789ABCDEF, 7), (2**64 - 1, 2**32 - 1)]:
        ctx.mask_bits(it, p, seed, out)
        torch.cuda.synchronize()
        ref = oracle.mask_bits(K, Hc, Wc, p, seed, it)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)
    ctx.close()


def test_lipschitz_parity(torch_dev):
    for K, s in [(8, 5), (100, 11), (3, 1), (17, 7)]:
        d = np.random.default_rng(K).standard_normal((K, s, s)).astype(np.float32)
        ctx = _ctx(1, K, s, s + 3, s + 3)
        L = ctx.lipschitz(_t(d, torch_dev))
        assert abs(L - oracle.lipschitz(d)) <= 1e-12 * L
        ctx.close()


@pytest.mark.parametrize("conv", ["half", "ss", "tmem"])
@pytest.mark.parametrize("shape", [(3, 5, 5, 70, 130), (2, 17, 11, 100, 100), (4, 8, 5, 32, 32),
                                   (1, 3, 1, 9, 65), (2, 6, 3, 129, 64), (1, 2, 9, 9, 9), (2, 130, 7, 41, 61),
                                   (1, 100, 11, 150, 40), (2, 400, 11, 20, 30), (1, 1024, 11, 12, 14)])
def test_residual_and_objective_parity(torch_dev, shape, conv, monkeypatch):
    """Dense pass r = Dz - x and the Eq.1 objective: TMA-fed SS tensor-core kernel (default where
    Hc*Wc % 4 == 0), TMEM-fed kernel, or SIMT (s < 5, W+s-1 < 32).  Shapes: k-splits (K=130),
    bands that end mid-tile, many bands (H=150)."""
    monkeypatch.setenv("CSC_CONV_PATH", conv)
    N, K, s, H, W = shape
    x, d, z = random_problem(100 + K, N, K, s, H, W, code_density=0.3)
    ctx = _ctx(N, K, s, H, W)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    lam = 0.7
    F = ctx.objective(xt, dt, zt, lam)
    r = _t(np.zeros_like(x), torch_dev)
    ctx.read_residual(r)
    import torch
    torch.cuda.synchronize()
    assert rel_err(r.cpu().numpy(), oracle.residual(x, d, z)) < TOL
    Fo = oracle.objective(x, d, z, lam)
    for a, b_ in zip(F, Fo):
        assert abs(a - b_) <= TOL * abs(b_)
    ctx.close()


def _assert_changed_set(x, d, z, zg, zo, m, lam, tau):
    """The set of codes the step changes is the oracle's, exactly, except where the pre-shrinkage
    value |w| = |z - tau c| lies within rounding distance of the threshold tau*lambda (there the
    decision is taken on a value the two sides round differently; reading T7)."""
    r = oracle.residual(x, d, z, dtype=np.float64)
    c = oracle.dtr(d, r, dtype=np.float64)
    w = z.astype(np.float64) - float(tau) * c
    kappa = float(tau) * lam
    amb = np.abs(np.abs(w) - kappa) <= 1e-4 * (kappa + float(tau) * np.abs(c)) + 1e-30
    mm = np.broadcast_to(m, z.shape)
    ch_g, ch_o = (zg != z) & mm, (zo != z) & mm
    diff = (ch_g != ch_o) & ~amb
    assert not diff.any(), f"{int(diff.sum())} codes change on one side only (of {int(mm.sum())} selected)"
    assert int((ch_g != ch_o).sum()) <= max(2, int(1e-4 * mm.sum()))


@pytest.mark.parametrize("K,s,H,W", [(100, 11, 256, 120), (130, 7, 20, 300), (8, 5, 32, 32), (400, 11, 30, 100),
                                     (17, 3, 9, 40)])
@pytest.mark.parametrize("p,mode", [(0.1, "entry"), (0.5, "entry"), (0.05, "sector8"), (1.0, "entry")])
def test_mask_selwords_bit_exact(torch_dev, K, s, H, W, p, mode):
    """The mask the tensor-core code step consumes (selection words, csc_mask_selwords) against the
    oracle's canonical mask, bit for bit, for several filter groups (K = 130, 400) and both modes."""
    import torch
    ctx = _ctx(1, K, s, H, W)
    if mode != "entry":
        ctx.set_mask_mode(mode)
    nkg, wper, wnc, KC = ctx.mask_selwords(0, p, 0)
    Hc, Wc = H + s - 1, W + s - 1
    out = torch.zeros(nkg * wper * Hc * Wc, dtype=torch.int32, device=torch_dev)
    for seed, it in [(7, 3), (2**64 - 1, 2**32 - 1)]:
        ctx.mask_selwords(it, p, seed, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32).reshape(nkg, wper, Hc * Wc)
        mb = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, it, mode=mode), K, Hc, Wc).reshape(K, -1)
        exp = np.zeros_like(got)
        for kg in range(nkg):
            kend = min(K, (kg + 1) * KC)
            for b in range(wper):
                for i in range(wnc):
                    k = kg * KC + b * wnc + i
                    if k < kend:
                        exp[kg, b] |= mb[k].astype(np.uint32) << np.uint32(i)
        assert np.array_equal(got, exp)
    ctx.close()


@pytest.mark.parametrize("path", ["half", "tc", "simt"])
@pytest.mark.parametrize("shape,p", [((3, 5, 5, 70, 130), 0.1), ((2, 17, 11, 100, 100), 0.2),
                                     ((4, 8, 5, 32, 32), 1.0), ((1, 9, 3, 33, 47), 0.5), ((2, 4, 11, 11, 11), 0.05),
                                     ((2, 130, 7, 20, 300), 0.1), ((1, 100, 11, 40, 11), 0.3), ((3, 16, 9, 61, 9), 1.0),
                                     ((2, 400, 11, 20, 30), 0.1), ((1, 1024, 11, 12, 14), 0.1)])
def test_code_step_parity(torch_dev, shape, p, path, monkeypatch):
    """Masked prox-gradient code step: tcgen05 dense-then-mask kernel or SIMT.  Shapes: several
    k-groups (K=130), tiles that wrap many short rows (Wc=21, 17), ragged plane tails, p=1 shortcut."""
    import torch
    monkeypatch.setenv("CSC_CODE_PATH", path)
    N, K, s, H, W = shape
    x, d, z = random_problem(200 + K, N, K, s, H, W, code_density=0.3)
    seed, it, lam = 12345, 3, 0.2
    ctx = _ctx(N, K, s, H, W)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    tau = ctx.code_step(xt, dt, zt, lam, p, seed, it, want_step=True)
    zg = zt.cpu().numpy()
    zo, tau_o = oracle.code_step(x, d, z, lam, 0.0, p, seed, it)
    assert abs(tau - tau_o) <= TOL_TAU * tau_o
    assert rel_err(zg, zo) < TOL
    Hc, Wc = H + s - 1, W + s - 1
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, it), K, Hc, Wc)
    for n in range(N):
        assert np.array_equal(zg[n][~m], z[n][~m])  # unsampled codes bit-identical (R2)
    _assert_changed_set(x, d, z, zg, zo, m, lam, tau_o)
    if ctx.variants & 32:
        # a3' (fp16-split code step): the code step leaves r' = r + D dz = D z_new - x in the residual cache
        r = torch.zeros_like(xt)
        ctx.read_residual(r)
        torch.cuda.synchronize()
        assert rel_err(r.cpu().numpy(), oracle.residual(x, d, zo)) < TOL
    # explicit step size
    zt2 = _t(z, torch_dev)
    ctx.invalidate()
    ctx.code_step(xt, dt, zt2, lam, p, seed, it, step_z=0.01)
    zo2, _ = oracle.code_step(x, d, z, lam, 0.01, p, seed, it)
    torch.cuda.synchronize()
    assert rel_err(zt2.cpu().numpy(), zo2) < TOL
    ctx.close()


@pytest.mark.parametrize("wg", ["h", "tf32", "simt"])
@pytest.mark.parametrize("shape", [(3, 5, 5, 70, 130), (2, 17, 11, 100, 100), (1, 3, 3, 9, 9), (2, 130, 5, 36, 40),
                                   (1, 8, 7, 26, 22), (2, 40, 11, 256, 56), (5, 24, 9, 48, 63), (1, 100, 11, 12, 300),
                                   (2, 400, 11, 20, 30), (1, 1024, 11, 12, 14), (3, 9, 3, 18, 22), (2, 33, 5, 41, 60)])
def test_filter_step_parity(torch_dev, shape, wg, monkeypatch):
    """Filter gradient g = Z^T r (tcgen05 kind::f16 3-term split kernel "h", the 3xTF32 kernel, or SIMT),
    exact line search, projection.
    Shapes cover several k-groups (K=130; K=400: four groups; K=1024: ten groups of 103 filters padded to
    112), one partial chunk per row (Wc < 32), chunks spanning rows (Wc < 64; odd Wc), a row of exactly
    one 64-position chunk, many bands, rows of 9-10 chunks, and Hc*Wc % 4 != 0 (TMA view impossible:
    SIMT path either way)."""
    import torch
    monkeypatch.setenv("CSC_WGRAD_PATH", wg)
    N, K, s, H, W = shape
    x, d, z = random_problem(300 + K, N, K, s, H, W, code_density=0.3)
    ctx = _ctx(N, K, s, H, W)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    Hc, Wc = H + s - 1, W + s - 1
    if wg == "h" and ctx.variants & 16 and (Hc * Wc) % 4 == 0:
        assert ctx.variants & 64  # the fp16-rate kernel is the one under test
    tau = ctx.filter_step(xt, dt, zt, want_step=True)
    g = torch.zeros(K * s * s, dtype=torch.float64, device=torch_dev)
    ctx.read_grad(g)
    torch.cuda.synchronize()
    do, tau_o, go, _ = oracle.filter_step(x, d, z)
    assert rel_err(g.cpu().numpy(), go.ravel()) < TOL
    assert abs(tau - tau_o) <= TOL_TAU * tau_o
    assert rel_err(dt.cpu().numpy(), do) < TOL
    assert (np.sqrt((dt.cpu().numpy().astype(np.float64) ** 2).sum(axis=(1, 2))) <= 1 + 1e-6).all()
    ctx.close()


def _trajectory(torch_dev, cfg, iters, p=None, check_every=1):
    import torch
    p = cfg.p if p is None else p
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    worst = {"z": 0.0, "d": 0.0, "F": 0.0, "tau_z": 0.0, "tau_d": 0.0}
    for t in range(1, iters + 1):
        F, taus = ctx.iterate(xt, dt, zt, cfg.lam, p, seed, t)
        it = oracle.iteration(x, d, z, cfg.lam, p, seed, t)
        z, d = it["z"], it["d"]
        if t % check_every == 0 or t == iters:
            torch.cuda.synchronize()
            errs = {"z": rel_err(zt.cpu().numpy(), z), "d": rel_err(dt.cpu().numpy(), d),
                    "F": abs(F[0] - it["F"][0]) / abs(it["F"][0]),
                    "tau_z": abs(taus[0] - it["tau_z"]) / it["tau_z"],
                    "tau_d": abs(taus[1] - it["tau_d"]) / max(it["tau_d"], 1e-30)}
            for k_, v in errs.items():
                worst[k_] = max(worst[k_], v)
            assert errs["z"] < TOL and errs["d"] < TOL and errs["F"] < TOL, (t, errs)
            # tau_z depends on d only (1e-6); along a trajectory tau_d is a function of the state (z, d),
            # which the bar holds to 1e-5 (reading T3); its one-step accuracy is
            # test_filter_step_parity's 1e-6
            assert errs["tau_z"] < TOL_TAU and errs["tau_d"] < TOL, (t, errs, worst)
    ctx.close()
    return worst


@pytest.mark.parametrize("dense", ["tc", "simt"])
def test_trajectory_tiny_50_iterations(torch_dev, dense, monkeypatch):
    """Config 1 (BASELINE.json configs[0]): 50 code+filter iterations, every iteration compared."""
    monkeypatch.setenv("CSC_DENSE_PATH", dense)
    w = _trajectory(torch_dev, CONFIGS["tiny"], 50)
    print(f"tiny dense={dense} worst", w)


def test_trajectory_ragged_multitile(torch_dev):
    """Several 64x64 tiles with ragged tails, s=11, p=0.2, 20 iterations."""
    cfg = CONFIGS["batch"].with_(name="ragged", N=3, K=12, H=70, W=135, p=0.2)
    _trajectory(torch_dev, cfg, 20)


@pytest.mark.parametrize("dense", ["tc", "simt"])
@pytest.mark.parametrize("p", [0.1, 1.0])
def test_trajectory_batch_config(torch_dev, p, dense, monkeypatch):
    """Config 2 (BASELINE.json configs[1]) at full size: first 5 iterations, every one compared,
    with the tensor-core (3xTF32) and the SIMT dense passes."""
    monkeypatch.setenv("CSC_DENSE_PATH", dense)
    w = _trajectory(torch_dev, CONFIGS["batch"], 5, p=p)
    print(f"batch p={p} dense={dense} worst", w)


def test_zero_codes_and_online_step(torch_dev):
    """SOCSC step (Alg.2): zero codes -> 10 masked code steps -> filter step -> objective."""
    import torch
    cfg = CONFIGS["online"].with_(K=24, N=3, H=40, W=44)
    x = make_images(cfg)
    d = make_filters(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt = _t(x, torch_dev), _t(d, torch_dev)
    zt = torch.full((cfg.N, cfg.K, cfg.Hc, cfg.Wc), 3.0, device=torch_dev)
    ctx.zero_codes(xt, zt)
    r = torch.zeros_like(xt)
    ctx.read_residual(r)
    torch.cuda.synchronize()
    assert not zt.any() and torch.equal(r, -xt)
    z = np.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), np.float32)
    for i in range(10):
        ctx.code_step(xt, dt, zt, cfg.lam, cfg.p, seed, i)
        z, _ = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, seed, i)
    ctx.filter_step(xt, dt, zt)
    d1, _, _, _ = oracle.filter_step(x, d, z)
    F = ctx.objective(xt, dt, zt, cfg.lam)
    Fo = oracle.objective(x, d1, z, cfg.lam)
    torch.cuda.synchronize()
    assert rel_err(zt.cpu().numpy(), z) < TOL
    assert rel_err(dt.cpu().numpy(), d1) < TOL
    assert abs(F[0] - Fo[0]) < TOL * Fo[0]
    ctx.close()


def test_empty_local_batch(torch_dev):
    """n_local = 0 (a rank with no images): steps are no-ops on codes, filters get a zero gradient."""
    import torch
    ctx = _ctx(0, 4, 3, 8, 8)
    d = _t(make_filters(CONFIGS["tiny"].with_(K=4, s=3)), torch_dev)
    d0 = d.clone()
    e = torch.zeros(0, device=torch_dev)
    ctx.code_step(e, d, e, 1.0, 0.5, 1, 1)
    ctx.filter_step(e, d, e)
    F = ctx.objective(e, d, e, 1.0)
    torch.cuda.synchronize()
    assert F == (0.0, 0.0, 0.0)
    assert torch.equal(d, d0)
    ctx.close()


def test_argument_errors(torch_dev):
    import torch
    import paper_1909_00145_b200 as pkg
    x, d, z = random_problem(1, 1, 2, 3, 8, 8)
    ctx = _ctx(1, 2, 3, 8, 8)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    z0 = zt.clone()
    for bad in [dict(p=0.0), dict(p=1.5), dict(lam=-1.0), dict(lam=float("nan"))]:
        kw = dict(lam=1.0, p=0.5)
        kw.update(bad)
        with pytest.raises(pkg.CSCError) as ei:
            ctx.code_step(xt, dt, zt, kw["lam"], kw["p"], 1, 1)
        assert ei.value.status == 1
    torch.cuda.synchronize()
    assert torch.equal(zt, z0)  # no side effects
    ctx.close()


@pytest.mark.slow
def test_full_size_sweep_config_sampled(torch_dev):
    """Config 3 (N=40, 256x256, K=100, s=11, p=0.1) in the launch configuration bench.py times:
    one full iteration on the GPU; the oracle checks sampled images for the code step (per-image
    independent), the full filter gradient / step and the objective."""
    import torch
    cfg = CONFIGS["sweep"]
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt, zt = _t(x, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    # iteration 1 from the initial state, codes first
    ctx.code_step(xt, dt, zt, cfg.lam, cfg.p, seed, 1)
    torch.cuda.synchronize()
    zg = zt.cpu().numpy()
    sample = [0, cfg.N - 1]
    zo, _ = oracle.code_step(x[sample], d, z[sample], cfg.lam, 0.0, cfg.p, seed, 1)
    assert rel_err(zg[sample], zo) < TOL
    # filter step + objective on the GPU's codes (all 40 images)
    tau = ctx.filter_step(xt, dt, zt, want_step=True)
    do, tau_o, _, _ = oracle.filter_step(x, d, zg)
    torch.cuda.synchronize()
    assert abs(tau - tau_o) <= TOL_TAU * tau_o
    assert rel_err(dt.cpu().numpy(), do) < TOL
    F = ctx.objective(xt, dt, zt, cfg.lam)
    Fo = oracle.objective(x, do, zg, cfg.lam)
    assert abs(F[0] - Fo[0]) <= TOL * Fo[0]
    ctx.close()


@pytest.mark.slow
def test_full_size_online_config_step():
    """Config 4 (BASELINE.json configs[3]) at full size: K=400 filters (4 filter groups in the
    tensor-core kernels), a mini-batch of 8 images 100x100, p=0.1 -- one SOCSC step (Alg.2,
    P:336-346; reading #14): zero codes, 10 masked code steps (mask t = 10 step + i), filter step,
    objective; codes, filters and F against the oracle."""
    import torch
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["online"]
    x = make_images(cfg, 0, cfg.N)
    d = make_filters(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt = _t(x, dev), _t(d, dev)
    zt = torch.empty((cfg.N, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    ctx.zero_codes(xt, zt)
    z = np.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), np.float32)
    step = 3
    for i in range(10):
        ctx.code_step(xt, dt, zt, cfg.lam, cfg.p, seed, 10 * step + i)
        z, _ = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, seed, 10 * step + i)
    ctx.filter_step(xt, dt, zt)
    d1, _, _, _ = oracle.filter_step(x, d, z)
    F = ctx.objective(xt, dt, zt, cfg.lam)
    Fo = oracle.objective(x, d1, z, cfg.lam)
    torch.cuda.synchronize()
    assert rel_err(zt.cpu().numpy(), z) < TOL
    assert rel_err(dt.cpu().numpy(), d1) < TOL
    assert abs(F[0] - Fo[0]) < TOL * Fo[0]
    ctx.close()


@pytest.mark.slow
def test_full_size_large_config_sampled():
    """Config 5 (BASELINE.json configs[4]) at full size on one B200: K=1024 filters (10 filter
    groups), 64 images 512x512, 71 GB of codes, p=0.1, in the launch configuration bench.py uses.
    Two iterations on the GPU; the code steps are checked on sampled images against the oracle
    (codes are independent per image given d), the filter step by properties that hold at any
    size: unit-ball filters and a decreasing objective."""
    import torch
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["large"]
    x = make_images(cfg)
    d = make_filters(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt = _t(x, dev), _t(d, dev)
    zt = torch.empty((cfg.N, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    ctx.zero_codes(xt, zt)
    sample = [0, cfg.N - 1]
    F_prev = 0.5 * float((x.astype(np.float64) ** 2).sum())
    z_s = np.zeros((len(sample), cfg.K, cfg.Hc, cfg.Wc), np.float32)
    for t in (1, 2):
        d_before = dt.cpu().numpy()
        ctx.code_step(xt, dt, zt, cfg.lam, cfg.p, seed, t)
        torch.cuda.synchronize()
        zo, _ = oracle.code_step(x[sample], d_before, z_s, cfg.lam, 0.0, cfg.p, seed, t)
        zg = torch.stack([zt[i] for i in sample]).cpu().numpy()
        assert rel_err(zg, zo) < TOL, (t, rel_err(zg, zo))
        z_s = zg
        ctx.filter_step(xt, dt, zt)
        F = ctx.objective(xt, dt, zt, cfg.lam)
        dn = np.sqrt((dt.cpu().numpy().astype(np.float64) ** 2).sum(axis=(1, 2)))
        assert (dn <= 1 + 1e-6).all()
        assert F[0] < F_prev, (t, F, F_prev)
        F_prev = F[0]
    del zt
    ctx.close()


def test_iterate_with_new_images_each_step(torch_dev):
    """csc_iterate with x_host: the residual cache is moved to the new images elementwise
    (r + x_old - x_new); 6 iterations on a different seeded batch each step match the oracle."""
    import torch
    cfg = CONFIGS["tiny"]
    p, lam = 0.5, cfg.lam
    d = make_filters(cfg)
    z = make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    x0 = make_images(cfg)
    xt, dt, zt = _t(x0, torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    for t in range(1, 7):
        xb = np.ascontiguousarray(make_images(cfg.with_(N=cfg.N), 0, cfg.N) * (1.0 + 0.1 * t)).astype(np.float32)
        xh = torch.from_numpy(xb).pin_memory()
        F, _ = ctx.iterate(xt, dt, zt, lam, p, seed, t, x_host=xh)
        it = oracle.iteration(xb, d, z, lam, p, seed, t)
        z, d = it["z"], it["d"]
        torch.cuda.synchronize()
        assert rel_err(zt.cpu().numpy(), z) < TOL, t
        assert rel_err(dt.cpu().numpy(), d) < TOL, t
        assert abs(F[0] - it["F"][0]) <= TOL * abs(it["F"][0]), t
    ctx.close()


def test_iterate_staged_double_buffered(torch_dev):
    """csc_stage_images + csc_iterate_staged: the next batch is staged on the copy stream while the
    current iteration runs; 5 iterations on different batches match the oracle, and an unstaged
    slot is refused."""
    import torch
    import paper_1909_00145_b200 as pkg
    cfg = CONFIGS["tiny"]
    p, lam = 0.5, cfg.lam
    d, z = make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt, zt = _t(make_images(cfg), torch_dev), _t(d, torch_dev), _t(z, torch_dev)
    batches = [np.ascontiguousarray(make_images(cfg) * (1.0 + 0.2 * t)).astype(np.float32) for t in range(5)]
    hosts = [torch.from_numpy(b).pin_memory() for b in batches]
    with pytest.raises(pkg.CSCError):
        ctx.iterate_staged(xt, dt, zt, lam, p, seed, 1, 1)
    ctx.stage_images(hosts[0], 0)
    for t in range(5):
        if t + 1 < 5:
            ctx.stage_images(hosts[t + 1], (t + 1) % 2)
        F, _ = ctx.iterate_staged(xt, dt, zt, lam, p, seed, t + 1, t % 2)
        it = oracle.iteration(batches[t], d, z, lam, p, seed, t + 1)
        z, d = it["z"], it["d"]
        torch.cuda.synchronize()
        assert rel_err(zt.cpu().numpy(), z) < TOL, t
        assert rel_err(dt.cpu().numpy(), d) < TOL, t
        assert abs(F[0] - it["F"][0]) <= TOL * abs(it["F"][0]), t
    ctx.close()


def test_iterate_staged_async_pipelined(torch_dev):
    """csc_iterate_staged_async returns the previous iteration's objective and step sizes while the next
    one is queued; csc_iterate_drain returns the last.  Same kernels as csc_iterate_staged: the sequence
    of (F, tau_z, tau_d), the codes and the filters are bit-identical to the synchronous calls, and the
    objectives match the oracle."""
    import torch
    cfg = CONFIGS["tiny"]
    p, lam, steps = 0.5, cfg.lam, 6
    seed = mask_seed(cfg)
    batches = [np.ascontiguousarray(make_images(cfg) * (1.0 + 0.2 * t)).astype(np.float32) for t in range(steps)]
    hosts = [torch.from_numpy(b).pin_memory() for b in batches]

    def run(use_async):
        ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
        xt = _t(make_images(cfg), torch_dev)
        dt, zt = _t(make_filters(cfg), torch_dev), _t(make_codes(cfg), torch_dev)
        out = []
        ctx.stage_images(hosts[0], 0)
        for t in range(steps):
            if t + 1 < steps:
                ctx.stage_images(hosts[t + 1], (t + 1) % 2)
            if use_async:
                r = ctx.iterate_staged_async(xt, dt, zt, lam, p, seed, t + 1, t % 2)
                assert (r is None) == (t == 0)
                if r is not None:
                    out.append(r)
            else:
                out.append(ctx.iterate_staged(xt, dt, zt, lam, p, seed, t + 1, t % 2))
        if use_async:
            r = ctx.iterate_drain()
            assert r is not None
            out.append(r)
            assert ctx.iterate_drain() is None
        torch.cuda.synchronize()
        res = (out, zt.cpu().numpy(), dt.cpu().numpy())
        ctx.close()
        return res

    sync_out, zs, ds = run(False)
    async_out, za, da = run(True)
    assert len(async_out) == steps
    assert async_out == sync_out
    assert np.array_equal(za, zs) and np.array_equal(da, ds)
    d, z = make_filters(cfg), make_codes(cfg)
    for t in range(steps):
        it = oracle.iteration(batches[t], d, z, lam, p, seed, t + 1)
        z, d = it["z"], it["d"]
        assert abs(async_out[t][0][0] - it["F"][0]) <= TOL * abs(it["F"][0]), t

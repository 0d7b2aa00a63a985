"""50-iteration parity on every BASELINE.json configuration (north_star: "codes, filters and
objective match within 1e-5 relative per iteration over 50 iterations on all five configs";
SURVEY.md §8(c) "Required agreement" and its per-config rule).

  config 1 (tiny)    tests/test_gpu_parity.py::test_trajectory_tiny_50_iterations (full z, live oracle)
  config 2 (batch)   test_trajectory_batch_50: full z, d, F, tau_z, tau_d every iteration, live oracle
  config 3 (sweep)   test_trajectory_sweep_golden: the committed oracle trajectory
                     (scripts/golden_trajectories.py, imports only oracle/ and synth/): d, F, tau_z,
                     tau_d, per-image norms and 2^14 sampled codes every iteration; per-(image, filter)
                     norms and 2^16 sampled codes at t in {1,2,5,10,25,50}; and the full codes of images
                     {0, 39} against the oracle's code step from the GPU's state at those t
  config 4 (online)  test_trajectory_online_golden: 50 SOCSC steps (Alg.2, reading #14) against the
                     committed oracle trajectory: d, F, the 10 tau_z and tau_d, per-(image, filter)
                     norms and 2^14 sampled codes every step
  config 5 (large)   test_large_config_sampled_50: 50 iterations; full codes of images {0, 63} against
                     the oracle's code step from the GPU's state at t in {1,2,5,10,25,50}; g, tau_d and F
                     of a 2-image sub-problem against the oracle's filter step / objective at t in {1, 50}

Tolerances: TOL = 1e-5 (norm-wise relative, reading R9/#16) for z, d, F, norms, r, g;
TOL_TAU = 1e-6 for the step sizes as functions of their inputs: tau_z every
iteration (it depends on d only), tau_d in the one-step checks from the GPU's own state.  Along a
trajectory tau_d is a function of the codes and filters, which the bar allows to differ by 1e-5, so the
trajectory value of tau_d is held to TOL (reading T3).
"""
import os

import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-5
TOL_TAU = 1e-6
CHECKPOINTS = (1, 2, 5, 10, 25, 50)
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def dev():
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


def _norms_n(zt):
    import torch
    a1 = torch.sum(zt.abs(), dim=(1, 2, 3), dtype=torch.float64)
    a2 = torch.sqrt(torch.sum(zt * zt, dim=(1, 2, 3), dtype=torch.float64))
    return a1.cpu().numpy(), a2.cpu().numpy()


def _norms_nk(zt):
    import torch
    a1 = torch.sum(zt.abs(), dim=(2, 3), dtype=torch.float64)
    a2 = torch.sqrt(torch.sum(zt * zt, dim=(2, 3), dtype=torch.float64))
    return a1.cpu().numpy(), a2.cpu().numpy()


def test_trajectory_batch_50(dev):
    """Config 2 (K=100, s=11, N=10 images 100x100, p=0.1) at full size: 50 iterations through
    csc_iterate, every one compared with the oracle's iteration in full."""
    import torch
    cfg = CONFIGS["batch"]
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt, zt = _t(x, dev), _t(d, dev), _t(z, dev)
    worst = {}
    for t in range(1, 51):
        d_prev = dt.cpu().numpy()
        F, taus = ctx.iterate(xt, dt, zt, cfg.lam, cfg.p, seed, t)
        it = oracle.iteration(x, d, z, cfg.lam, cfg.p, seed, t)
        z, d = it["z"], it["d"]
        torch.cuda.synchronize()
        zg = zt.cpu().numpy()
        e = {"z": rel_err(zg, z), "d": rel_err(dt.cpu().numpy(), d),
             "F": abs(F[0] - it["F"][0]) / abs(it["F"][0]),
             "tau_z": abs(taus[0] - it["tau_z"]) / it["tau_z"],
             "tau_d": abs(taus[1] - it["tau_d"]) / max(it["tau_d"], 1e-30)}
        if t in CHECKPOINTS:
            # the filter step from the GPU's own state (codes after this iteration's code step, the
            # filters before it): the line-search step to 1e-6
            d1, tau_o, _, _ = oracle.filter_step(x, d_prev, zg)
            e["tau_d_step"] = abs(taus[1] - tau_o) / tau_o
            e["d_step"] = rel_err(dt.cpu().numpy(), d1)
            assert e["tau_d_step"] < TOL_TAU and e["d_step"] < TOL, (t, e)
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        assert e["z"] < TOL and e["d"] < TOL and e["F"] < TOL, (t, e)
        assert e["tau_z"] < TOL_TAU and e["tau_d"] < TOL, (t, e)
    print("batch worst", worst)
    ctx.close()


def _check_code_step_from_gpu_state(x_s, d_prev, z_prev_s, z_now_s, lam, p, seed, t):
    """The GPU's codes of a sample of images after iteration t against the oracle's code step
    from the GPU's own state before it (codes are independent per image given d)."""
    zo, _ = oracle.code_step(x_s, d_prev, z_prev_s, lam, 0.0, p, seed, t)
    err = rel_err(z_now_s, zo)
    assert err < TOL, (t, err)
    return err


def _subproblem_check(x, d_prev, zt, sample, cfg, dev):
    """The filter step and the objective of a sub-problem made of a few images (the GPU's codes after
    this iteration's code step, the filters before its filter step) on a fresh context of that size, in
    the same launch configuration family, against the oracle: g, d and F to 1e-5, tau_d to 1e-6."""
    import torch
    x2 = np.ascontiguousarray(x[sample])
    z2 = torch.stack([zt[i] for i in sample]).contiguous()
    d2 = _t(d_prev, dev)
    c2 = _ctx(len(sample), cfg.K, cfg.s, cfg.H, cfg.W)
    x2t = _t(x2, dev)
    tau2 = c2.filter_step(x2t, d2, z2, want_step=True)
    g2 = torch.zeros(cfg.K * cfg.s * cfg.s, dtype=torch.float64, device=dev)
    c2.read_grad(g2)
    F2 = c2.objective(x2t, d2, z2, cfg.lam)
    torch.cuda.synchronize()
    z2n = z2.cpu().numpy()
    do, tau_o, go, _ = oracle.filter_step(x2, d_prev, z2n)
    Fo = oracle.objective(x2, do, z2n, cfg.lam)
    e = {"sub_g": rel_err(g2.cpu().numpy(), go.ravel()), "sub_d": rel_err(d2.cpu().numpy(), do),
         "sub_tau_d": abs(tau2 - tau_o) / tau_o, "sub_F": abs(F2[0] - Fo[0]) / Fo[0]}
    c2.close()
    return e


def test_trajectory_sweep_golden(dev):
    """Config 3 (K=100, s=11, N=40 images 256x256, p=0.1; the benched configuration, through
    csc_iterate as bench.py times it): 50 iterations against the committed oracle trajectory."""
    import torch
    path = os.path.join(GOLDEN, "traj_sweep_p0.1.npz")
    gd = np.load(path)
    cfg = CONFIGS["sweep"]
    p = float(gd["p"])
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    assert int(gd["seed"]) == seed
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt, zt = _t(x, dev), _t(d, dev), _t(z, dev)
    idx_s = torch.from_numpy(gd["idx_s"]).to(dev)
    idx_b = torch.from_numpy(gd["idx_b"]).to(dev)
    sample = [0, cfg.N - 1]
    worst = {}
    ck = list(gd["ck_t"])
    for t in range(1, int(gd["iters"]) + 1):
        if t in CHECKPOINTS:
            d_prev = dt.cpu().numpy()
            z_prev = torch.stack([zt[i] for i in sample]).cpu().numpy()
        F, taus = ctx.iterate(xt, dt, zt, cfg.lam, p, seed, t)
        torch.cuda.synchronize()
        i = t - 1
        n1, n2 = _norms_n(zt)
        zflat = zt.view(-1)
        e = {"d": rel_err(dt.cpu().numpy(), gd["d"][i]),
             "F": abs(F[0] - gd["F"][i, 0]) / gd["F"][i, 0],
             "tau_z": abs(taus[0] - gd["tau_z"][i]) / gd["tau_z"][i],
             "tau_d": abs(taus[1] - gd["tau_d"][i]) / gd["tau_d"][i],
             "zn1": rel_err(n1, gd["zn1"][i]), "zn2": rel_err(n2, gd["zn2"][i]),
             "zs": rel_err(zflat[idx_s].cpu().numpy(), gd["zs"][i])}
        if t in CHECKPOINTS:
            j = ck.index(t)
            a1, a2 = _norms_nk(zt)
            e["znk1"] = rel_err(a1, gd["ck_znk1"][j])
            e["znk2"] = rel_err(a2, gd["ck_znk2"][j])
            e["zb"] = rel_err(zflat[idx_b].cpu().numpy(), gd["ck_zb"][j])
            z_now = torch.stack([zt[i2] for i2 in sample]).cpu().numpy()
            e["z_step"] = _check_code_step_from_gpu_state(x[sample], d_prev, z_prev, z_now, cfg.lam, p, seed, t)
        if t in (1, 50):
            e.update(_subproblem_check(x, d_prev, zt, sample, cfg, dev))
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        for k in ("d", "F", "zn1", "zn2", "zs", "znk1", "znk2", "zb", "tau_d", "sub_g", "sub_d", "sub_F"):
            if k in e:
                assert e[k] < TOL, (t, k, e)
        assert e["tau_z"] < TOL_TAU, (t, e)
        if "sub_tau_d" in e:
            assert e["sub_tau_d"] < TOL_TAU, (t, e)
    print("sweep worst", worst)
    ctx.close()


def test_trajectory_online_golden(dev):
    """Config 4 (K=400 filters 11x11, mini-batches of 8 images 100x100, p=0.1): 50 SOCSC steps
    (Alg.2; reading #14: fresh batch 8s..8s+7, z = 0, 10 masked code steps with mask
    iterations 10 s + i, projected-gradient filter step, objective over the batch) against the
    committed oracle trajectory."""
    import torch
    gd = np.load(os.path.join(GOLDEN, "traj_online.npz"))
    cfg = CONFIGS["online"]
    n_inner = int(gd["n_inner"])
    seed = mask_seed(cfg)
    assert int(gd["seed"]) == seed
    nb = cfg.N
    ctx = _ctx(nb, cfg.K, cfg.s, cfg.H, cfg.W)
    dt = _t(make_filters(cfg), dev)
    xt = torch.empty((nb, cfg.H, cfg.W), dtype=torch.float32, device=dev)
    zt = torch.empty((nb, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    idx_s = torch.from_numpy(gd["idx_s"]).to(dev)
    worst = {}
    for s in range(int(gd["steps"])):
        xt.copy_(torch.from_numpy(make_images(cfg, nb * s, nb)))
        ctx.zero_codes(xt, zt)
        taus = [ctx.code_step(xt, dt, zt, cfg.lam, cfg.p, seed, n_inner * s + i, want_step=True)
                for i in range(n_inner)]
        tau_d = ctx.filter_step(xt, dt, zt, want_step=True)
        F = ctx.objective(xt, dt, zt, cfg.lam)
        torch.cuda.synchronize()
        a1, a2 = _norms_nk(zt)
        e = {"d": rel_err(dt.cpu().numpy(), gd["d"][s]),
             "F": abs(F[0] - gd["F"][s, 0]) / gd["F"][s, 0],
             "tau_z": float(np.max(np.abs(np.array(taus) - gd["tau_z"][s]) / gd["tau_z"][s])),
             "tau_d": abs(tau_d - gd["tau_d"][s]) / gd["tau_d"][s],
             "znk1": rel_err(a1, gd["znk1"][s]), "znk2": rel_err(a2, gd["znk2"][s]),
             "zs": rel_err(zt.view(-1)[idx_s].cpu().numpy(), gd["zs"][s])}
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        for k in ("d", "F", "znk1", "znk2", "zs", "tau_d"):
            assert e[k] < TOL, (s, k, e)
        assert e["tau_z"] < TOL_TAU, (s, e)
    print("online worst", worst)
    ctx.close()


@pytest.mark.slow
def test_large_config_sampled_50():
    """Config 5 (K=1024, s=11, N=64 images 512x512, 71 GB of codes on one B200, p=0.1) in the launch
    configuration bench.py uses: 50 iterations through csc_iterate.  SURVEY.md §8(c) rule for the
    configurations too large for a full oracle trajectory: the full codes of images {0, 63} against
    the oracle's code step from the GPU's state at t in {1,2,5,10,25,50}; g, tau_d and F of a 2-image
    sub-problem (those images, the GPU's codes and filters) against the oracle's filter step and
    objective at t in {1, 50}."""
    import torch
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["large"]
    x = make_images(cfg)
    d = make_filters(cfg)
    seed = mask_seed(cfg)
    sample = [0, cfg.N - 1]
    ctx = _ctx(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W)
    xt, dt = _t(x, dev), _t(d, dev)
    zt = torch.empty((cfg.N, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    ctx.zero_codes(xt, zt)
    worst = {}
    F_prev = None
    for t in range(1, 51):
        if t in CHECKPOINTS:
            d_prev = dt.cpu().numpy()
            z_prev = torch.stack([zt[i] for i in sample]).cpu().numpy()
        F, taus = ctx.iterate(xt, dt, zt, cfg.lam, cfg.p, seed, t)
        dn = np.sqrt((dt.cpu().numpy().astype(np.float64) ** 2).sum(axis=(1, 2)))
        assert (dn <= 1 + 1e-6).all()
        if F_prev is not None:
            assert F[0] < F_prev, (t, F, F_prev)
        F_prev = F[0]
        if t in CHECKPOINTS:
            z_now = torch.stack([zt[i] for i in sample]).cpu().numpy()
            e = _check_code_step_from_gpu_state(x[sample], d_prev, z_prev, z_now, cfg.lam, cfg.p, seed, t)
            worst["z_step"] = max(worst.get("z_step", 0.0), e)
        if t in (1, 50):
            e = _subproblem_check(x, d_prev, zt, sample, cfg, dev)
            for k, v in e.items():
                worst[k] = max(worst.get(k, 0.0), v)
            assert e["sub_g"] < TOL and e["sub_d"] < TOL and e["sub_F"] < TOL, (t, e)
            assert e["sub_tau_d"] < TOL_TAU, (t, e)
    print("large worst", worst)
    del zt
    ctx.close()

"""Write the golden trajectories of BASELINE.json configs 3 and 4 with the CPU oracle.

    python scripts/golden_trajectories.py sweep  [--iters 50] [--p 0.1]
    python scripts/golden_trajectories.py online [--steps 50]

TEST INFRASTRUCTURE.  Imports only oracle/ (the plain CPU implementation) and synth/ (the seeded
input recipe); nothing here comes from the CUDA path.  The GPU parity tests
(tests/test_gpu_trajectories.py) replay the same iterations through the C ABI and compare every
iteration with what is stored here ("Required agreement"; DESIGN.md §2 "golden
trajectories").

Config 3 ("sweep", K=100, s=11, N=40, 256x256, p=0.1): 50 SBCSC iterations (Alg.1,
PAPER.md:287-301) from the initial state.  Stored per iteration t = 1..50: the filters d^t (fp32,
in full), F^t (F, 1/2||r||^2, lam||z||_1), tau_z^t, tau_d^t, per-image ||z_n||_1, ||z_n||_2 and
non-zero counts, and the codes at a fixed seeded sample of 2^14 coordinates; at t in
{1, 2, 5, 10, 25, 50} also the per-(image, filter) norms and 2^16 sampled coordinates.  The full
code tensor (1.13 GB per iteration) is not stored (reading G1).

Config 4 ("online", K=400, 8 images 100x100 per mini-batch, p=0.1): 50 SOCSC steps (Alg.2,
PAPER.md:333-347; reading #14): for step s = 0..49 the mini-batch holds images 8s..8s+7 of the
seeded stream, the codes start at 0, 10 masked code steps use mask iterations t = 10 s + i, then one
projected-gradient filter step and the objective over the batch.  Stored per step: d (fp32, in
full), F, the 10 tau_z, tau_d, per-(image, filter) norms of the batch codes, and 2^14 sampled code
coordinates.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import CONFIGS, ROOT_SEED, make_codes, make_filters, make_images, mask_seed  # noqa: E402

CHECKPOINTS = (1, 2, 5, 10, 25, 50)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def sample_index(cfg_index: int, total: int, count: int, salt: int) -> np.ndarray:
    """A fixed seeded sample of flat code indices (sorted, without repetition)."""
    rng = np.random.default_rng(np.random.SeedSequence([ROOT_SEED, cfg_index, 99, salt]))
    return np.sort(rng.choice(total, size=min(count, total), replace=False)).astype(np.int64)


def norms_n(z):
    zf = z.reshape(z.shape[0], -1).astype(np.float64)
    return np.abs(zf).sum(axis=1), np.sqrt((zf * zf).sum(axis=1)), (zf != 0).sum(axis=1)


def norms_nk(z):
    zf = z.reshape(z.shape[0], z.shape[1], -1).astype(np.float64)
    return np.abs(zf).sum(axis=2), np.sqrt((zf * zf).sum(axis=2))


def sweep(iters: int, p: float, out: str):
    cfg = CONFIGS["sweep"]
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    total = z.size
    idx_s = sample_index(cfg.index, total, 1 << 14, 1)
    idx_b = sample_index(cfg.index, total, 1 << 16, 2)
    rec = {k: [] for k in ("d", "F", "tau_z", "tau_d", "zn1", "zn2", "nnz", "zs")}
    ck = {k: [] for k in ("t", "znk1", "znk2", "zb")}
    t0 = time.time()
    for t in range(1, iters + 1):
        it = oracle.iteration(x, d, z, cfg.lam, p, seed, t)
        z, d = it["z"], it["d"]
        n1, n2, nz = norms_n(z)
        rec["d"].append(d.copy())
        rec["F"].append(np.array(it["F"], np.float64))
        rec["tau_z"].append(it["tau_z"])
        rec["tau_d"].append(it["tau_d"])
        rec["zn1"].append(n1)
        rec["zn2"].append(n2)
        rec["nnz"].append(nz)
        rec["zs"].append(z.ravel()[idx_s].copy())
        if t in CHECKPOINTS:
            a1, a2 = norms_nk(z)
            ck["t"].append(t)
            ck["znk1"].append(a1)
            ck["znk2"].append(a2)
            ck["zb"].append(z.ravel()[idx_b].copy())
        print(f"sweep t={t} F={it['F'][0]:.6f} tau_z={it['tau_z']:.6g} tau_d={it['tau_d']:.6g} "
              f"nnz={nz.sum() / total:.4f} {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(
        out, config="sweep", p=p, iters=iters, lam=cfg.lam, seed=np.uint64(seed), idx_s=idx_s, idx_b=idx_b,
        d=np.stack(rec["d"]).astype(np.float32), F=np.stack(rec["F"]), tau_z=np.array(rec["tau_z"]),
        tau_d=np.array(rec["tau_d"]), zn1=np.stack(rec["zn1"]), zn2=np.stack(rec["zn2"]),
        nnz=np.stack(rec["nnz"]), zs=np.stack(rec["zs"]).astype(np.float32), ck_t=np.array(ck["t"]),
        ck_znk1=np.stack(ck["znk1"]), ck_znk2=np.stack(ck["znk2"]), ck_zb=np.stack(ck["zb"]).astype(np.float32),
        oracle_threads=oracle.num_threads(), oracle_seconds=time.time() - t0)


def online(steps: int, out: str, n_inner: int = 10):
    cfg = CONFIGS["online"]
    d = make_filters(cfg)
    seed = mask_seed(cfg)
    nb = cfg.N
    total = nb * cfg.K * cfg.Hc * cfg.Wc
    idx_s = sample_index(cfg.index, total, 1 << 14, 1)
    rec = {k: [] for k in ("d", "F", "tau_z", "tau_d", "znk1", "znk2", "zs")}
    t0 = time.time()
    for s in range(steps):
        x = make_images(cfg, nb * s, nb)
        z = make_codes(cfg, nb)
        taus = []
        for i in range(n_inner):
            z, tz = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, seed, n_inner * s + i)
            taus.append(tz)
        d, tau_d, _, _ = oracle.filter_step(x, d, z)
        F = oracle.objective(x, d, z, cfg.lam)
        a1, a2 = norms_nk(z)
        rec["d"].append(d.copy())
        rec["F"].append(np.array(F, np.float64))
        rec["tau_z"].append(np.array(taus))
        rec["tau_d"].append(tau_d)
        rec["znk1"].append(a1.astype(np.float32))
        rec["znk2"].append(a2.astype(np.float32))
        rec["zs"].append(z.ravel()[idx_s].copy())
        print(f"online step={s} F={F[0]:.6f} tau_d={tau_d:.6g} {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(
        out, config="online", p=cfg.p, steps=steps, n_inner=n_inner, lam=cfg.lam, seed=np.uint64(seed),
        idx_s=idx_s, d=np.stack(rec["d"]).astype(np.float32), F=np.stack(rec["F"]),
        tau_z=np.stack(rec["tau_z"]), tau_d=np.array(rec["tau_d"]), znk1=np.stack(rec["znk1"]),
        znk2=np.stack(rec["znk2"]), zs=np.stack(rec["zs"]).astype(np.float32),
        oracle_threads=oracle.num_threads(), oracle_seconds=time.time() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["sweep", "online"])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    if a.which == "sweep":
        out = a.out or os.path.join(GOLDEN, f"traj_sweep_p{a.p:g}.npz")
        sweep(a.iters, a.p, out)
    else:
        out = a.out or os.path.join(GOLDEN, "traj_online.npz")
        online(a.steps, out)
    print("wrote", out)


if __name__ == "__main__":
    main()

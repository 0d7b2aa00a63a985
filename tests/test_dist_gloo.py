"""Multi-rank host logic on CPU (world_size 2, gloo): the image sharding and the
ncclUniqueId broadcast used by the NCCL path, and the sharded iteration: the
filter gradient, ||Zg||^2 and the objective parts summed over ranks (what the
library all-reduces) reproduce the single-process oracle iteration exactly in
the fp64 build (codes are data-independent per image; the
mask is identical on every rank, reading R5)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1909_00145_b200 import dist as cdist
from synth import CONFIGS, make_codes, make_filters, make_images, mask_seed


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_iteration(x, d, z, lam, p, seed, t, allreduce):
    """One SBCSC iteration with this rank's images; allreduce(np.ndarray) sums over ranks."""
    z1, tau_z = oracle.code_step(x, d, z, lam, 0.0, p, seed, t, dtype=np.float64)
    r = oracle.residual(x, d, z1, dtype=np.float64)
    g = allreduce(oracle.filter_grad(r, z1, dtype=np.float64))
    zg = oracle.residual(None, g, z1, dtype=np.float64)
    zg2 = allreduce(np.array([np.sum(zg * zg)]))[0]
    tau_d = float(np.sum(g * g) / zg2) if zg2 > 0 else 0.0
    e = d - tau_d * g
    nrm = np.sqrt((e * e).sum(axis=(1, 2), keepdims=True))
    d1 = e / np.maximum(1.0, nrm)
    F = oracle.objective(x, d1, z1, lam, dtype=np.float64)
    parts = allreduce(np.array([F[1], F[2]]))
    return z1, d1, tau_z, tau_d, parts


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ncclUniqueId broadcast: every rank gets rank 0's bytes
        nid = cdist.broadcast_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        cfg = CONFIGS["tiny"].with_(N=5)  # odd N: uneven shards 2 / 3
        n0, n1 = cdist.shard(cfg.N, world, rank)
        x = make_images(cfg, n0, n1 - n0).astype(np.float64)
        d = make_filters(cfg).astype(np.float64)
        z = make_codes(cfg, n1 - n0).astype(np.float64)

        def allreduce(a):
            tt = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(tt)
            return tt.numpy()

        out = []
        for t in (1, 2, 3):
            z, d, tau_z, tau_d, parts = _sharded_iteration(x, d, z, cfg.lam, cfg.p, mask_seed(cfg), t, allreduce)
            out.append((tau_z, tau_d, parts.copy()))
        zs = [None] * world
        dist.all_gather_object(zs, (n0, z))
        if rank == 0:
            q.put({"ids": ids, "d": d, "z": zs, "iters": out})
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in range(0, 20):
        for world in (1, 2, 4, 8):
            blocks = [cdist.shard(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        cdist.shard(4, 2, 2)


def test_gloo_world2_sharded_iteration_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    assert res["ids"][0] == res["ids"][1] and len(res["ids"][0]) == 128

    cfg = CONFIGS["tiny"].with_(N=5)
    x = make_images(cfg).astype(np.float64)
    d = make_filters(cfg).astype(np.float64)
    z = make_codes(cfg).astype(np.float64)
    for t, (tau_z, tau_d, parts) in zip((1, 2, 3), res["iters"]):
        it = oracle.iteration(x, d, z, cfg.lam, cfg.p, mask_seed(cfg), t, dtype=np.float64)
        z, d = it["z"], it["d"]
        assert abs(tau_z - it["tau_z"]) <= 1e-12 * it["tau_z"]
        assert abs(tau_d - it["tau_d"]) <= 1e-12 * it["tau_d"]
        assert abs(parts[0] - it["F"][1]) <= 1e-12 * it["F"][1]
        assert abs(parts[1] - it["F"][2]) <= 1e-12 * max(it["F"][2], 1e-300)
    assert np.max(np.abs(res["d"] - d)) <= 1e-12
    zsh = np.concatenate([zz for _, zz in sorted(res["z"], key=lambda a: a[0])])
    assert np.max(np.abs(zsh - z)) <= 1e-12

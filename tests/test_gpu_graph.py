"""CUDA-graph capture of a SOCSC step through the C ABI (include/csc.h "CUDA GRAPHS"; SURVEY.md §7 hard
part 7: the online configuration is launch-bound, so its inner loop is replayed as one graph).

One step of Alg.2 (reading #14): zero codes, 10 masked code steps (mask iterations
10 s + i), the projected-gradient filter step.  Captured once on the context's stream, replayed on
fresh mini-batches with the step's mask iterations supplied through the device-side offset
(csc_set_iter_offset), it must produce the same codes and filters as the same calls issued eagerly on a
second context (same kernels in the same order: bit-identical), and the eager run matches the oracle."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_filters, make_images, mask_seed
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu


def test_socsc_step_graph_replay():
    import torch
    import paper_1909_00145_b200 as pkg
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["online"].with_(K=48, N=4, H=40, W=44)
    seed = mask_seed(cfg)
    n_inner = 10
    s_cap = torch.cuda.Stream(dev)
    s_eag = torch.cuda.Stream(dev)
    cg = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_cap)
    ce = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_eag)
    d0 = make_filters(cfg)
    xg = torch.empty((cfg.N, cfg.H, cfg.W), device=dev)
    zg = torch.empty((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev)
    dg = torch.from_numpy(d0).to(dev)

    def socsc(ctx, x, d, z, step):
        ctx.zero_codes(x, z)
        for i in range(n_inner):
            ctx.code_step(x, d, z, cfg.lam, cfg.p, seed, n_inner * step + i)
        ctx.filter_step(x, d, z)

    off = torch.zeros(1, dtype=torch.int32, device=dev)
    cg.set_iter_offset(off)

    # warm-up (first launches configure the kernels), then capture step 0's sequence
    xg.copy_(torch.from_numpy(make_images(cfg, 0, cfg.N)))
    with torch.cuda.stream(s_cap):
        socsc(cg, xg, dg, zg, 0)
    torch.cuda.synchronize()
    dg.copy_(torch.from_numpy(d0))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s_cap):
        socsc(cg, xg, dg, zg, 0)
    torch.cuda.synchronize()
    # replay on fresh mini-batches: step s uses mask iterations 10 s + i through the device offset
    dg.copy_(torch.from_numpy(d0))
    de = torch.from_numpy(d0).to(dev)
    xe = torch.empty_like(xg)
    ze = torch.empty_like(zg)
    d_or = d0.copy()
    for b in range(3):
        xb = torch.from_numpy(make_images(cfg, cfg.N * (b + 1), cfg.N))
        step = b + 1
        xg.copy_(xb)
        xe.copy_(xb)
        off.fill_(n_inner * step)
        torch.cuda.synchronize()
        graph.replay()
        with torch.cuda.stream(s_eag):
            socsc(ce, xe, de, ze, step)
        torch.cuda.synchronize()
        assert torch.equal(zg, ze), b
        assert torch.equal(dg, de), b
        # and the eager step against the oracle
        xn = xb.numpy()
        z = np.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), np.float32)
        for i in range(n_inner):
            z, _ = oracle.code_step(xn, d_or, z, cfg.lam, 0.0, cfg.p, seed, n_inner * step + i)
        d_or, _, _, _ = oracle.filter_step(xn, d_or, z)
        assert rel_err(ze.cpu().numpy(), z) < 1e-5, b
        assert rel_err(de.cpu().numpy(), d_or) < 1e-5, b
    cg.close()
    ce.close()


def test_iteration_graph_replay_matches_iterate():
    """A whole SBCSC iteration (Alg.1: csc_code_step, csc_filter_step, csc_objective_enqueue) captured once
    and replayed with the mask iteration in the device offset gives the same codes, filters and objective
    as csc_iterate called eagerly on a second context (bench.py's timed loop)."""
    import torch
    import paper_1909_00145_b200 as pkg
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["batch"].with_(K=40, N=3, H=44, W=40, p=0.2)
    seed = mask_seed(cfg)
    x = torch.from_numpy(make_images(cfg)).to(dev)
    d0 = make_filters(cfg)
    s_g, s_e = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cg = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_g)
    ce = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_e)
    dg, de = torch.from_numpy(d0).to(dev), torch.from_numpy(d0).to(dev)
    zg = torch.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev)
    ze = torch.zeros_like(zg)
    off = torch.zeros(1, dtype=torch.int32, device=dev)
    cg.set_iter_offset(off)
    torch.cuda.synchronize()
    # two eager iterations on both contexts (the steady state the graph is captured in)
    for it in (1, 2):
        Fg = cg.iterate(x, dg, zg, cfg.lam, cfg.p, seed, it)[0]
        Fe = ce.iterate(x, de, ze, cfg.lam, cfg.p, seed, it)[0]
        assert Fg == Fe
    torch.cuda.synchronize()

    def body():
        cg.code_step(x, dg, zg, cfg.lam, cfg.p, seed, 0)
        cg.filter_step(x, dg, zg)
        cg.objective_enqueue(x, dg, zg)

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s_g):
        # warm the capture path once eagerly at iteration 3
        off.fill_(3)
        body()
        Fg3 = cg.objective_read(cfg.lam)
    Fe3 = ce.iterate(x, de, ze, cfg.lam, cfg.p, seed, 3)[0]
    assert Fg3 == Fe3
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s_g):
        body()
    for it in (4, 5, 6):
        with torch.cuda.stream(s_g):
            off.fill_(it)
        torch.cuda.synchronize()
        with torch.cuda.stream(s_g):  # replay on the context's stream (objective_read syncs that stream)
            graph.replay()
        Fg = cg.objective_read(cfg.lam)
        Fe = ce.iterate(x, de, ze, cfg.lam, cfg.p, seed, it)[0]
        torch.cuda.synchronize()
        assert Fg == Fe, it
        assert torch.equal(zg, ze), it
        assert torch.equal(dg, de), it
    cg.close()
    ce.close()


def test_streaming_step_graph_replay():
    """csc_load_staged captured with the iteration (csc_code_step, csc_filter_step, csc_objective_enqueue):
    one graph per staging slot, replayed on batches staged from pinned host memory (external event
    nodes wait for each slot's latest copy), produces the same objectives, codes and filters as eager
    csc_iterate_staged calls on a second context (bit-identical)."""
    import torch
    import paper_1909_00145_b200 as pkg
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    cfg = CONFIGS["tiny"]
    seed, p, lam, steps = mask_seed(cfg), 0.5, cfg.lam, 6
    batches = [np.ascontiguousarray(make_images(cfg) * (1.0 + 0.2 * t)).astype(np.float32) for t in range(steps + 3)]
    hosts = [torch.from_numpy(b).pin_memory() for b in batches]
    s_cap, s_eag = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cg = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_cap)
    ce = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_eag)
    d0 = make_filters(cfg)

    def fresh():
        return (torch.from_numpy(make_images(cfg)).to(dev), torch.from_numpy(d0).to(dev),
                torch.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev))

    # eager reference: csc_iterate_staged on batches 0 .. steps-1 after one warm-up step on batch 0
    xe, de, ze = fresh()
    ref = []
    with torch.cuda.stream(s_eag):
        ce.stage_images(hosts[0], 0)
        ce.iterate_staged(xe, de, ze, lam, p, seed, 1, 0)
        for t in range(steps):
            ce.stage_images(hosts[t], (t + 1) % 2)
            ref.append(ce.iterate_staged(xe, de, ze, lam, p, seed, t + 2, (t + 1) % 2)[0])
    torch.cuda.synchronize()

    # graphs: the same warm-up step eagerly, then one capture per slot, replayed with the step's iteration
    xg, dg, zg = fresh()
    off = torch.zeros(1, dtype=torch.int32, device=dev)
    cg.set_iter_offset(off)
    with torch.cuda.stream(s_cap):
        cg.stage_images(hosts[0], 0)
        cg.iterate_staged(xg, dg, zg, lam, p, seed, 1, 0)
    torch.cuda.synchronize()
    state = [t.clone() for t in (xg, dg, zg)]
    graphs = []
    for sl in (0, 1):
        with torch.cuda.stream(s_cap):
            cg.stage_images(hosts[0], sl)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s_cap):
            cg.load_staged(xg, sl)
            cg.code_step(xg, dg, zg, lam, p, seed, 0)
            cg.filter_step(xg, dg, zg)
            cg.objective_enqueue(xg, dg, zg)
        graphs.append(g)
    torch.cuda.synchronize()
    for t_, s_ in zip((xg, dg, zg), state):  # capture ran nothing; restore anyway
        t_.copy_(s_)
    torch.cuda.synchronize()
    got = []
    with torch.cuda.stream(s_cap):
        for t in range(steps):
            cg.stage_images(hosts[t], (t + 1) % 2)
            off.fill_(t + 2)
            graphs[(t + 1) % 2].replay()
            got.append(cg.objective_read(lam))
    torch.cuda.synchronize()
    assert got == ref
    assert torch.equal(zg, ze) and torch.equal(dg, de)
    cg.close()
    ce.close()

"""Development aid: which part of a captured iteration diverges from the eager one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00145_b200 as pkg
from synth import CONFIGS, make_filters, make_images, mask_seed

torch.cuda.set_device(0)
dev = torch.device("cuda:0")
cfg = CONFIGS["batch"].with_(K=40, N=3, H=44, W=40, p=0.2)
seed = mask_seed(cfg)
x = torch.from_numpy(make_images(cfg)).to(dev)
d0 = make_filters(cfg)
for parts in (("code",), ("code", "filter"), ("code", "filter", "obj")):
    s_g, s_e = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cg = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_g)
    ce = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=s_e)
    dg, de = torch.from_numpy(d0).to(dev), torch.from_numpy(d0).to(dev)
    zg = torch.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev)
    ze = torch.zeros_like(zg)
    off = torch.zeros(1, dtype=torch.int32, device=dev)
    cg.set_iter_offset(off)
    torch.cuda.synchronize()
    for it in (1, 2):
        cg.iterate(x, dg, zg, cfg.lam, cfg.p, seed, it)
        ce.iterate(x, de, ze, cfg.lam, cfg.p, seed, it)
    torch.cuda.synchronize()

    def body(ctx, dd, zz, it):
        if "code" in parts: ctx.code_step(x, dd, zz, cfg.lam, cfg.p, seed, it)
        if "filter" in parts: ctx.filter_step(x, dd, zz)
        if "obj" in parts: ctx.objective_enqueue(x, dd, zz)
        else: ctx.objective(x, dd, zz, cfg.lam) if False else None

    with torch.cuda.stream(s_g):
        off.fill_(3)
        body(cg, dg, zg, 0)
    with torch.cuda.stream(s_e):
        body(ce, de, ze, 3)
    torch.cuda.synchronize()
    print(parts, "eager it3 equal z", torch.equal(zg, ze), "d", torch.equal(dg, de))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s_g):
        body(cg, dg, zg, 0)
    for it in (4, 5):
        with torch.cuda.stream(s_g):
            off.fill_(it)
        torch.cuda.synchronize()
        graph.replay()
        with torch.cuda.stream(s_e):
            body(ce, de, ze, it)
        torch.cuda.synchronize()
        print(parts, it, "z equal", torch.equal(zg, ze), float((zg - ze).abs().max()), "d equal", torch.equal(dg, de),
              float((dg - de).abs().max()))
    cg.close(); ce.close()

import time, torch, sys
sys.path.insert(0, '.')
import paper_1909_00145_b200 as pkg
from synth import CONFIGS, make_images, make_filters, mask_seed
cfg = CONFIGS["sweep"]; dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream)
x = torch.from_numpy(make_images(cfg)).to(dev); d = torch.from_numpy(make_filters(cfg)).to(dev)
z = torch.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev)
ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0, stream=stream)
seed = mask_seed(cfg); off = torch.zeros(1, dtype=torch.int32, device=dev); ctx.set_iter_offset(off)
def body():
    ctx.code_step(x, d, z, cfg.lam, cfg.p, seed, 0); ctx.filter_step(x, d, z); ctx.objective_enqueue(x, d, z)
for i in range(3):
    off.fill_(i + 1); body(); ctx.objective_read(cfg.lam)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    body()
xh = torch.from_numpy(make_images(cfg)).pin_memory()
ctx.stage_images(xh, 0); ctx.load_staged(x, 0); torch.cuda.synchronize()
it = 10
def run(mode, n=20):
    global it
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if mode >= 1: ctx.stage_images(xh, 0)
    for i in range(n):
        it += 1
        if mode >= 1 and i + 1 < n: ctx.stage_images(xh, (i + 1) % 2)
        if mode >= 2: ctx.load_staged(x, i % 2)
        off.fill_(it); g.replay(); ctx.objective_read(cfg.lam)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
for mode in (0, 1, 2, 0, 1, 2):
    if mode >= 1:
        pass
    ms = run(mode)
    print("mode", mode, "ms/step %.3f" % ms, flush=True)

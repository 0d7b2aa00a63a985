"""Development aid: filter-gradient error of the tensor-core path vs the oracle for several shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_1909_00145_b200 as pkg
from synth import random_problem
from tests.conftest import rel_err
torch.cuda.set_device(0)
for shape in [(3, 5, 5, 70, 130), (2, 17, 11, 100, 100), (2, 40, 11, 256, 56)]:
    N, K, s, H, W = shape
    x, d, z = random_problem(300 + K, N, K, s, H, W, code_density=0.3)
    ctx = pkg.Context(N, K, s, H, W, device=0)
    dev = torch.device("cuda:0")
    xt, dt, zt = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, d, z)]
    tau = ctx.filter_step(xt, dt, zt, want_step=True)
    g = torch.zeros(K * s * s, dtype=torch.float64, device=dev)
    ctx.read_grad(g)
    torch.cuda.synchronize()
    do, tau_o, go, _ = oracle.filter_step(x, d, z)
    print(os.environ.get("CSC_WGRAD_PATH", "tc"), os.environ.get("CSC_WG_CPT", "8"), shape,
          f"g {rel_err(g.cpu().numpy(), go.ravel()):.2e} tau {abs(tau - tau_o) / tau_o:.2e} d {rel_err(dt.cpu().numpy(), do):.2e}"
          f" |tau g|/|d| {tau_o * np.linalg.norm(go) / np.linalg.norm(d):.2f}", flush=True)
    ctx.close()

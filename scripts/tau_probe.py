"""tau_d error probe: the tiny trajectory state after the first code step, filter step through each
dense-pass variant (CSC_CONV_PATH / CSC_DENSE_PATH), relative error of tau_d against the oracle."""
import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

def run(env_kv):
    code = r'''
import numpy as np, torch, json, sys
sys.path.insert(0, %r)
import oracle, paper_1909_00145_b200 as pkg
from synth import CONFIGS, make_images, make_filters, make_codes, mask_seed
out = []
for name in ["tiny", "batch"]:
    cfg = CONFIGS[name]
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    seed = mask_seed(cfg)
    for t in (1, 2, 3):
        z, _ = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, seed, t)
        ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
        dev = torch.device("cuda:0")
        xt, dt, zt = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, d, z)]
        tau = ctx.filter_step(xt, dt, zt, want_step=True)
        d1, tau_o, g, zg2 = oracle.filter_step(x, d, z)
        out.append((name, t, abs(tau - tau_o) / tau_o))
        ctx.close()
        d = d1
print(json.dumps(out))
''' % ROOT
    env = dict(os.environ); env.update(env_kv)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    return r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]

for kv in [{}, {"CSC_CONV_PATH": "ss"}, {"CSC_CONV_PATH": "tmem"}, {"CSC_DENSE_PATH": "simt"}]:
    print(kv, run(kv), flush=True)

"""Per-iteration trace of a BASELINE.json configuration (paper_1909_00145_b200/trace.py): writes the CSV
(iter, F, fit, l1, nnz, tau_z, tau_d, ms_code, ms_filter, ms_obj, ms_iter) for `--iters` iterations of
Alg.1 from z = 0 on the seeded synthetic workload of synth.CONFIGS.

    python scripts/trace_run.py --config sweep --iters 100 --out profiles/r02_trace_sweep.csv
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sweep")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--nvtx", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_1909_00145_b200 as pkg
    from paper_1909_00145_b200.trace import run_traced
    from synth import CONFIGS, make_filters, make_images, mask_seed
    cfg = CONFIGS[a.config]
    if a.p is not None:
        cfg = cfg.with_(p=a.p)
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(make_images(cfg)).to(dev)
    d = torch.from_numpy(make_filters(cfg)).to(dev)
    z = torch.zeros((cfg.N, cfg.K, cfg.Hc, cfg.Wc), device=dev)
    ctx = pkg.Context(cfg.N, cfg.K, cfg.s, cfg.H, cfg.W, device=0)
    ctx.set_nvtx(a.nvtx)
    tr = run_traced(ctx, x, d, z, cfg.lam, cfg.p, mask_seed(cfg), a.iters, start_iter=1)
    tr.write_csv(a.out)
    r0, r1 = tr.rows[0], tr.rows[-1]
    print(f"{a.config} p={cfg.p}: {len(tr)} iterations, F {r0['F']:.6g} -> {r1['F']:.6g}, nnz {r1['nnz']}, "
          f"median ms/iter {sorted(tr.column('ms_iter'))[len(tr) // 2]:.3f}")
    ctx.close()


if __name__ == "__main__":
    main()

"""bench.py -- CSC iterations/s on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config sweep] [--p 0.1] [--impl ours|reference]

A step is one SBCSC outer iteration (Alg.1) over the whole
hot path (every SURVEY.md §8(a) row): Philox mask + masked prox-gradient code
step, filter gradient + exact line search + unit-ball projection, Eq.1
objective -- through the C ABI call csc_iterate.

Default workload: config 3 "sweep" (BASELINE.json configs[2]) at p = 0.1:
K=100 filters 11x11, N=40 images 256x256, codes 100x266x266 per image (1.13 GB,
larger than the 126 MB L2, so no L2 flush is needed between steps).  It is the
largest configuration whose iteration fits one GPU in a few ms and the one
SURVEY.md §8(d) designates for HBM claims; configs[1] ("batch", 48 MB of codes)
is L2-resident and is reported with --config batch.  See DESIGN.md §6.

Multi-GPU (torchrun, one process per GPU): the N images are sharded across
ranks (strong scaling of the fixed problem); the filter gradient and the
objective parts are all-reduced with NCCL inside the library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
SMS = 148
FP32_LANES_PER_SM = 128


FALLBACK_BF16_TFLOPS = 1590.0
TF32_PER_BF16 = 1.1 / 2.25   # guide's nominal dense ratio (B200_PROFILING.md)


def _peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return (float(pk["hbm_gbs"]), float(pk.get("sm_max_mhz", 1965.0)), float(pk["bf16_tflops"]),
                "measured")
    except Exception:
        return FALLBACK_HBM_GBS, 1965.0, FALLBACK_BF16_TFLOPS, "fallback"


TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")


def _traffic():
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel class
    from the committed ncu --set full captures (profiles/traffic.json, written by
    scripts/ncu_traffic.py from profiles/*_ncu_*.txt); {} if absent."""
    try:
        with open(TRAFFIC_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


# kernel classes timed with CUDA events inside the timed region (kernel_rooflines reads these)
ROOFLINE_CLASSES = ("conv", "wgrad", "code_step", "admm", "bcd")


def kernel_rooflines(prof, cfg, nl, steps, variants, solver="prox", filter_solver="pg"):
    """Per kernel class: algorithmic work per launch / measured average launch time vs its roofs.
    Algorithmic units: dense pass / filter gradient 2*N*K*s^2*H*W FLOP and a read of
    all codes (4*N*K*Hc*Wc B); masked code step: sector-model bytes.  Tensor peaks: the measured
    bf16 peak (fp16 split kernels) or x 0.489 (nominal tf32/bf16, 3xTF32 kernels), / 3 products.
    "bound" is the roof with the larger fraction (the one the kernel is closest to)."""
    hbm_gbs, sm_max_mhz, bf16_tflops, kind = _peaks()
    fp32_peak = SMS * FP32_LANES_PER_SM * 2 * sm_max_mhz * 1e6 / 1e12
    tf32_peak = bf16_tflops * TF32_PER_BF16
    dense_flops = 2.0 * nl * cfg.K * cfg.s * cfg.s * cfg.H * cfg.W
    codes = nl * cfg.K * cfg.Hc * cfg.Wc
    traffic = _traffic()
    out = {}

    def two_roofs(kernel, avg, tpeak, tnote):
        t_ach = dense_flops / (avg / 1e3) / 1e12
        h_ach = 4.0 * codes / (avg / 1e3) / 1e9
        tensor = {"bound": "tensor", "achieved": t_ach, "peak": tpeak, "unit": "TFLOP/s", "peak_note": tnote,
                  "frac": t_ach / tpeak}
        hbm = {"bound": "hbm", "achieved": h_ach, "peak": hbm_gbs, "unit": "GB/s", "frac": h_ach / hbm_gbs,
               "peak_note": f"{kind} copy bandwidth (MEASURED_PEAKS.json)", "bytes_model": "4 N K Hc Wc (codes read once)"}
        best = dict(tensor if tensor["frac"] >= hbm["frac"] else hbm)
        best["kernel"] = kernel
        best["other_roof"] = hbm if best["bound"] == "tensor" else tensor
        return best

    for name, (ms, n) in prof.items():
        if n == 0:
            continue
        avg = ms / n
        if name == "conv":
            if variants & 16:
                out[name] = two_roofs("conv_h_kernel (tcgen05 kind::f16, 3-term fp16 split, TMA-fed SS)", avg,
                                      bf16_tflops / 3.0, f"{kind} bf16/fp16 {bf16_tflops:.0f} TF/s / 3 products")
            elif variants & 1:
                nm = "conv_ss_kernel (tcgen05 3xTF32, TMA-fed SS)" if variants & 8 else \
                    "conv_tc_kernel (tcgen05 3xTF32, TMEM A)"
                out[name] = two_roofs(nm, avg, tf32_peak / 3.0,
                                      f"{kind} bf16 {bf16_tflops:.0f} TF/s x {TF32_PER_BF16:.3f} (tf32/bf16 nominal) / 3")
            else:
                out[name] = {"kernel": "conv_fwd_kernel (SIMT FP32)", "bound": "alu",
                             "achieved": dense_flops / (avg / 1e3) / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
                             "peak_note": f"148 SMs x 128 FP32 lanes x 2 x {sm_max_mhz:.0f} MHz (derived)"}
        elif name == "wgrad" and variants & 64:
            out[name] = two_roofs("wgrad_h_kernel (tcgen05 kind::f16 3-term split, TMA z + TMEM im2col(r))", avg,
                                  bf16_tflops / 3.0, f"{kind} bf16/fp16 {bf16_tflops:.0f} TF/s / 3 products")
        elif name == "wgrad" and variants & 2:
            out[name] = two_roofs("wgrad_tc_kernel (tcgen05 3xTF32, TMA z + TMEM im2col(r))", avg, tf32_peak / 3.0,
                                  f"{kind} bf16 {bf16_tflops:.0f} TF/s x {TF32_PER_BF16:.3f} (tf32/bf16 nominal) / 3")
        elif name == "wgrad":
            out[name] = {"kernel": "wgrad_kernel (SIMT FP32)", "bound": "alu",
                         "achieved": dense_flops / (avg / 1e3) / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
                         "peak_note": f"148 SMs x 128 FP32 lanes x 2 x {sm_max_mhz:.0f} MHz (derived)"}
        elif name == "bcd":
            # Gram blocks C_kk = sum_n Z_nk^T Z_nk in fp64 dominate: N K H W (M^2/2 + M/2) fp64 FMA per sweep
            # (upper triangle incl. the diagonal tiles), against the fp64 FMA rate
            M = cfg.s * cfg.s
            nt = (M + 3) // 4
            lagged = cfg.H > cfg.s - 1 and cfg.W > cfg.s - 1
            if filter_solver == "surrogate" and lagged:  # lag-structured pair Grams
                fma = nl * (cfg.K * (cfg.K + 1) / 2) * (2 * cfg.s - 1) ** 2 * cfg.Hc * cfg.Wc
            elif filter_solver == "surrogate":  # direct pair Grams, full 4x4 tiles
                fma = nl * cfg.H * cfg.W * (cfg.K * (cfg.K + 1) / 2) * 16.0 * nt * nt
            elif lagged:  # lag-structured Gram: (2s-1)^2 lags x Hc x Wc
                fma = nl * cfg.K * (2 * cfg.s - 1) ** 2 * cfg.Hc * cfg.Wc
            else:
                fma = nl * cfg.K * cfg.H * cfg.W * 16.0 * nt * (nt + 1) / 2
            fp64_peak = SMS * 64 * 2 * sm_max_mhz * 1e6 / 1e12
            out[name] = {"kernel": "bcd_lag_kernel / bcd_gram_kernel + per-filter kernels (fp64, csc_bcd.cu)",
                         "bound": "alu",
                         "achieved": 2.0 * fma / (ms / steps / 1e3) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                         "peak_note": f"148 SMs x 64 FP64 lanes x 2 x {sm_max_mhz:.0f} MHz (derived, DESIGN.md §11)",
                         "flop_model": "Gram FMAs x 2 per sweep: lag-structured N K (2s-1)^2 Hc Wc (H, W > s-1), else "
                                       "N K H W 16 ceil(M/4)(ceil(M/4)+1)/2; whole class time"}
        elif name == "code_step" and solver == "admm":
            # ADMM mode: code_h_kernel in plain mode writes the dense correlation D^T e
            out[name] = two_roofs("code_h_kernel plain mode (dense D^T e for the ADMM operator)", avg,
                                  bf16_tflops / 3.0, f"{kind} bf16/fp16 {bf16_tflops:.0f} TF/s / 3 products")
            for rr_ in (out[name], out[name]["other_roof"]):
                if rr_["bound"] == "hbm":
                    rr_["bytes_model"] = "4 N K Hc Wc (dense correlation written once)"
        elif name == "admm":
            # vector / gather / expansion kernels of one ADMM step (10 x 5 CG), bytes per step:
            # 50 expansions (4C dense write + 12 Mc), 51 gathers (sector-model read of C + 8 Mc),
            # 50 CG steps (24 Mc), 10 updates (28 Mc), init + final scatter (2 x (sector C + 8 Mc))
            mcn = cfg.p * codes
            sect = 4.0 * (1.0 - (1.0 - cfg.p) ** 8) * codes
            step_bytes = (50 * (4.0 * codes + 12 * mcn) + 51 * (sect + 8 * mcn) + 50 * 24 * mcn + 10 * 28 * mcn
                          + 2 * (sect + 8 * mcn))
            per_step_ms = ms / steps
            out[name] = {"kernel": "ADMM vector kernels (expand, gather, cg_step, update; csc_admm.cu)",
                         "bound": "hbm", "achieved": step_bytes / (per_step_ms / 1e3) / 1e9, "peak": hbm_gbs,
                         "unit": "GB/s", "peak_note": f"{kind} copy bandwidth (MEASURED_PEAKS.json)",
                         "bytes_model": "per step: 50(4C+12Mc) + 51(4C(1-(1-p)^8)+8Mc) + 1200Mc + 280Mc + 2(...)"
                                        ", C = N K Hc Wc, Mc = p C; achieved = model bytes / class time per step"}
        elif name == "code_step":
            sector_bytes = 8.0 * (1.0 - (1.0 - cfg.p) ** 8) * codes + 12.0 * nl * cfg.H * cfg.W
            out[name] = {"kernel": ("code_h_kernel (tcgen05 kind::f16 3-term split, dense-then-mask, TMA code slices)" if variants & 32 else "code_tc_kernel (tcgen05 3xTF32 dense-then-mask)") if variants & 4
                         else "code_step_kernel (SIMT masked prox step)", "bound": "hbm",
                         "achieved": sector_bytes / (avg / 1e3) / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                         "peak_note": f"{kind} copy bandwidth (MEASURED_PEAKS.json)",
                         "bytes_model": "sector: 8(1-(1-p)^8) N K Hc Wc + 12 N H W"}
        else:
            continue
        r = out[name]
        r["frac"] = r["achieved"] / r["peak"]
        r["avg_launch_ms"] = avg
        r["launches_per_step"] = n / steps
        r["ms_per_step"] = ms / steps
        tr = traffic.get(name, {}).get(cfg.name)
        r["traffic"] = tr["bytes_per_launch"] if tr else None
        if tr:
            r["traffic_source"] = tr["source"]
    return out


class ClockSampler:
    """SM clocks and throttle reasons sampled every 5 ms DURING the timed region (B200_PROFILING.md
    clocks line), through NVML in a background thread; nvidia-smi -lms 20 as a fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._thr = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            h = None
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    if h is not None:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.samples.append((sm, rs))
                except Exception:
                    pass
                self._stop.wait(0.005)

        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def stop(self):
        if self._thr is None:
            return None
        self._stop.set()
        self._thr.join(timeout=2)
        if not self.samples:
            return None
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, 5 ms"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_step(cfg, x, d, z, t, oracle):
    """One step of the workload on the oracle: an SBCSC iteration (Alg.1), or for the online
    configuration an SOCSC step (Alg.2, reading #14: z = 0, 10 code steps, filter step, objective)."""
    if cfg.online:
        import numpy as np
        z = np.zeros_like(z)
        for i in range(cfg.n_inner):
            z, _ = oracle.code_step(x, d, z, cfg.lam, 0.0, cfg.p, _seed(cfg), cfg.n_inner * t + i)
        d, _, _, _ = oracle.filter_step(x, d, z)
        oracle.objective(x, d, z, cfg.lam)
        return d, z
    it = oracle.iteration(x, d, z, cfg.lam, cfg.p, _seed(cfg), t)
    return it["d"], it["z"]


def _seed(cfg):
    from synth import mask_seed
    return mask_seed(cfg)


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on the host cores (rank 0 only; the other ranks
    exit without work).  Each step is a bounded sample of the workload: the same iteration on
    --ref-images of the N images with every host thread busy (the oracle's passes are parallel over
    image rows, the code step over (image, filter)), its time scaled by N / sample to the full
    workload (the work is linear in the number of images)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import oracle
    from synth import config_by_name, make_codes, make_filters, make_images
    cfg = config_by_name(args.config, args.p)
    n_img = max(1, min(cfg.N, args.ref_images))
    sub = cfg.with_(N=n_img)
    x, d, z = make_images(sub), make_filters(sub), make_codes(sub)
    for t in range(1, args.warmup + 1):
        d, z = _oracle_step(cfg, x, d, z, t, oracle)
    times = []
    for t in range(args.warmup + 1, args.warmup + 1 + args.steps):
        t0 = time.perf_counter()
        d, z = _oracle_step(cfg, x, d, z, t, oracle)
        times.append(time.perf_counter() - t0)
    per_sample = sum(times) / len(times)
    per_full = per_sample * cfg.N / n_img
    value = 1.0 / per_full
    cores = oracle.num_threads()
    line = {
        "impl": "reference", "metric": "csc_iterations_per_s", "value": value, "unit": "it/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_full * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 state, f64 sums (CPU oracle)", "data": "synthetic", "config": _config_dict(cfg, ws),
        "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "cpu_model": _cpu_model(), "kind": "oracle",
                         "sample": f"{args.steps} steps, each the full step on {n_img} of {cfg.N} images with "
                                   f"{cores} threads ({per_sample:.2f} s), scaled x{cfg.N / n_img:g}"},
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "fits_in_driver_run": True,
    }
    print(json.dumps(line), flush=True)


def _config_dict(cfg, ws):
    return {"workload": f"{cfg.name} (BASELINE.json configs[{cfg.index - 1}]) p={cfg.p:g}",
            "K": cfg.K, "s": cfg.s, "N": cfg.N, "H": cfg.H, "W": cfg.W, "p": cfg.p, "lambda": cfg.lam,
            "codes_bytes": 4 * cfg.N * cfg.K * cfg.Hc * cfg.Wc, "global_batch": cfg.N,
            "parallelism": f"dp{ws} (images sharded)",
            "l2": "inputs larger than L2 (no flush)" if 4 * cfg.N * cfg.K * cfg.Hc * cfg.Wc > 126e6 * 2
            else "L2 flushed between steps"}


def _cpu_baseline(cfg):
    """The oracle on the host cores (rank 0, N = 1 only): ONE full step of the benched workload (all N
    images; M = 1, no extrapolation), every host thread."""
    import oracle
    from synth import make_codes, make_filters, make_images
    x, d, z = make_images(cfg), make_filters(cfg), make_codes(cfg)
    t0 = time.perf_counter()
    _oracle_step(cfg, x, d, z, 1, oracle)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": "it/s", "cores": oracle.num_threads(), "cpu_model": _cpu_model(),
            "kind": "oracle",
            "sample": f"M = 1 full step (step 1) on all {cfg.N} images, {dt:.1f} s, {oracle.num_threads()} threads"}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_00145_b200 as pkg
    from paper_1909_00145_b200 import dist as cdist
    from synth import config_by_name, make_codes, make_filters, make_images, mask_seed

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = config_by_name(args.config, args.p)
    n0, n1 = cdist.shard(cfg.N, ws, rank)
    nl = n1 - n0
    x_np = make_images(cfg, n0, nl)
    d_np = make_filters(cfg)
    seed = mask_seed(cfg)
    x = torch.from_numpy(x_np).to(dev)
    d = torch.from_numpy(d_np).to(dev)
    z = torch.zeros((nl, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    nccl_id = cdist.broadcast_nccl_id(device=dev) if ws > 1 else None
    torch.cuda.synchronize()
    # the library's stream: a dedicated stream (a CUDA graph cannot be captured on the legacy default
    # stream); torch's work of the timed loop (L2 flush, events) goes to the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = pkg.Context(nl, cfg.K, cfg.s, cfg.H, cfg.W, world=ws, rank=rank, device=local, stream=stream,
                      nccl_id=nccl_id)
    if args.step_rule != "lipschitz":
        ctx.set_step_rule(args.step_rule)
    if args.mask != "entry":
        ctx.set_mask_mode(args.mask)
    l2_flush = None
    if 4 * cfg.N * cfg.K * cfg.Hc * cfg.Wc <= 2 * 126e6:
        l2_flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    admm = args.code_solver == "admm"
    bcd = args.filter_solver == "bcd"
    sur = args.filter_solver == "surrogate"
    if sur:
        ctx.surrogate_reset()

    def step(it, x_host=None):
        """One outer iteration: csc_iterate (prox code step + projected-gradient filter step), or with
        --code-solver admm / --filter-solver bcd the paper's ADMM code update (csc_code_step_admm) /
        projected block-coordinate filter update (csc_filter_step_bcd), then the objective."""
        if not admm and not bcd and not sur:
            return ctx.iterate(x, d, z, cfg.lam, cfg.p, seed, it, x_host=x_host)
        if x_host is not None:
            x.copy_(x_host, non_blocking=True)
            ctx.invalidate()
        if admm:
            ctx.code_step_admm(x, d, z, cfg.lam, cfg.p, seed, it)
        else:
            ctx.code_step(x, d, z, cfg.lam, cfg.p, seed, it)
        if bcd:
            ctx.filter_step_bcd(x, d, z)
        elif sur:
            ctx.surrogate_update(x, z)
            ctx.filter_step_surrogate(d)
        else:
            ctx.filter_step(x, d, z)
        return ctx.objective(x, d, z, cfg.lam), None

    # mask iterations: iter + *off (csc_set_iter_offset); 0 for the eager calls, the step's iteration for
    # the graph replays
    off = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.set_iter_offset(off)
    it = 0
    for _ in range(args.warmup):
        it += 1
        step(it)
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs.  The prox / projected-gradient iteration (code step,
    # filter step, objective pass) is captured once as a CUDA graph and replayed every step, the step's
    # mask iteration written to the device offset first; each step then reads F (csc_objective_read,
    # host sync) as csc_iterate does.  The kernel durations of the roofline come from a second capture of
    # the same iteration with CUDA events around the long kernels (external event-record nodes), replayed
    # as many times right after the timed region: the event nodes cost ~4% of a step, so they are kept
    # out of the timed graph.  The other solvers (--code-solver admm, --filter-solver bcd|surrogate)
    # allocate on first use and run eagerly, with events on the long kernels inside the timed loop.
    use_graph = not (admm or bcd or sur) and not args.no_graph
    graph = graph_ev = None
    graph_launches = 0
    if use_graph:
        def body():
            ctx.code_step(x, d, z, cfg.lam, cfg.p, seed, 0)
            ctx.filter_step(x, d, z)
            ctx.objective_enqueue(x, d, z)
        it += 1
        off.fill_(it)
        ctx.profile_enable(True, classes=ROOFLINE_CLASSES)  # one eager profiled run fills the event pool
        body()
        ctx.objective_read(cfg.lam)
        ctx.profile_read()
        ctx.profile_enable(False)
        graph = torch.cuda.CUDAGraph()
        lc0 = ctx.launch_count
        with torch.cuda.graph(graph, stream=stream):
            body()
        graph_launches = ctx.launch_count - lc0
        ctx.profile_enable(True, classes=ROOFLINE_CLASSES)
        graph_ev = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_ev, stream=stream):
            body()
        torch.cuda.synchronize()
    else:
        ctx.profile_enable(True, classes=ROOFLINE_CLASSES)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count
    t_total = 0.0
    objs = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        it += 1
        if l2_flush is not None:
            l2_flush.fill_(float(it))
        if graph is not None:
            off.fill_(it)
            ev0.record(stream)
            graph.replay()
            ev1.record(stream)
            obj = ctx.objective_read(cfg.lam)
        else:
            ev0.record(stream)
            obj, taus = step(it)
            ev1.record(stream)
        ev1.synchronize()
        t_total += ev0.elapsed_time(ev1)
        objs.append(obj[0])
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = (graph_launches * args.steps) if graph is not None else ctx.launch_count - l0
    if graph_ev is not None:
        # the kernel-timing replays: the same iteration with event nodes around the long kernels
        for _ in range(args.steps):
            it += 1
            if l2_flush is not None:
                l2_flush.fill_(float(it))
            off.fill_(it)
            graph_ev.replay()
            ctx.objective_read(cfg.lam)
            ctx.profile_sample()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    off.fill_(0)
    tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    value = args.steps / (t_ms / 1e3)
    if rank == 0:
        print(f"[bench] timed region: {value:.2f} it/s, {t_ms / args.steps:.4f} ms/step", file=sys.stderr, flush=True)

    # ---- the per-class breakdown of every kernel class (untimed: events on every launch)
    ctx.profile_enable(True)
    tb0 = torch.cuda.Event(enable_timing=True)
    tb1 = torch.cuda.Event(enable_timing=True)
    tb0.record(stream)
    for _ in range(args.steps):
        it += 1
        if l2_flush is not None:
            l2_flush.fill_(float(it))
        step(it)
    tb1.record(stream)
    tb1.synchronize()
    prof_all = ctx.profile_read()
    t_prof = tb0.elapsed_time(tb1)
    ctx.profile_enable(False)

    # ---- e2e: same iteration through the C ABI with the step's images uploaded from pinned host memory.
    # Hot path: double-buffered -- step i+1's images are staged (async H2D on the library's copy stream)
    # before step i runs, so every step's transfer is inside the timed region but overlaps compute; and
    # pipelined -- csc_iterate_staged_async enqueues step i and returns step i-1's objective (the 80-B
    # D2H read of every step is inside the timed region, the device never waits for the host).
    x_host = torch.from_numpy(x_np).pin_memory()
    barrier()
    torch.cuda.synchronize()
    staged = not (admm or bcd or sur)
    if staged:  # one untimed staged iteration (the first call allocates the staging buffers and copy stream)
        it += 1
        ctx.stage_images(x_host, 0)
        ctx.iterate_staged(x, d, z, cfg.lam, cfg.p, seed, it, 0)
        torch.cuda.synchronize()
    # (A graph per staging slot of csc_load_staged + the iteration, with external event nodes for the
    # copies, measured slower end to end than these pipelined eager calls: 496 vs 530 it/s at config 3.)
    barrier()
    t0 = time.perf_counter()
    if staged:
        ctx.stage_images(x_host, 0)
    n_obj = 0
    for i in range(args.steps):
        it += 1
        if l2_flush is not None:
            l2_flush.fill_(float(it))
        if staged:
            # pipelined: enqueue this step, read the previous step's objective (80 B D2H per step), then start
            # the next step's upload (it overlaps this step)
            if ctx.iterate_staged_async(x, d, z, cfg.lam, cfg.p, seed, it, i % 2) is not None:
                n_obj += 1
            if i + 1 < args.steps:
                ctx.stage_images(x_host, (i + 1) % 2)
        else:
            step(it, x_host=x_host)
    if staged:
        n_obj += ctx.iterate_drain() is not None
        assert n_obj == args.steps
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / (float(te.item()) / 1e3)

    if rank == 0:
        step_ms = t_ms / args.steps
        rl = kernel_rooflines(prof, cfg, nl, args.steps, ctx.variants, args.code_solver, args.filter_solver)
        dom = max(rl, key=lambda k: rl[k]["ms_per_step"])
        kernels = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                       "share": v[0] / max(t_prof, 1e-9)} for k, v in prof_all.items()}
        line = {
            "metric": "csc_iterations_per_s", "value": value, "unit": "it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 state; fp16 3-term split products on the tensor cores, fp32 accumulate, fp64 reductions",
            "data": "synthetic",
            "config": dict(_config_dict(cfg, ws), code_solver=args.code_solver, filter_solver=args.filter_solver,
                           step_rule=args.step_rule, mask=args.mask, cuda_graph=graph is not None),
            "roofline": dict(rl[dom], dominant_class=dom),
            "kernel_rooflines": rl,
            "kernels": kernels,
            "kernels_note": "every class, from a second profiled pass of the same number of steps (events on every "
                            "launch); the timed region times only the roofline classes " + "/".join(ROOFLINE_CLASSES),
            "objective_last": objs[-1] if objs else None,
            "e2e": {"value": e2e_value, "unit": "it/s", "h2d_bytes_per_step": 4 * nl * cfg.H * cfg.W,
                    "d2h_bytes_per_step": 80},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = _cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


def run_online(args):
    """Config 4 (BASELINE.json configs[3]) as the paper's SOCSC step (Alg.2; reading #14): a
    fresh mini-batch of 8 images per step (images 8 s .. 8 s + 7 of the seeded stream, sharded over the
    ranks), codes reset to zero, 10 masked code steps with mask iterations 10 s + i, the projected-gradient
    filter step and the objective over the batch.  The zero / code / filter sequence is captured once as a
    CUDA graph on the library's stream and replayed every step (the mask iterations come from a
    device-side offset, csc_set_iter_offset); the objective (a host read) follows each replay."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_00145_b200 as pkg
    from paper_1909_00145_b200 import dist as cdist
    from synth import config_by_name, make_filters, make_images, mask_seed

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = config_by_name(args.config, args.p)
    nb, n_inner = cfg.N, cfg.n_inner
    n0, n1 = cdist.shard(nb, ws, rank)
    nl = n1 - n0
    n_steps = args.warmup + 2 + 2 * args.steps
    pool = np.stack([make_images(cfg, nb * st + n0, nl) for st in range(n_steps)])
    pool_dev = torch.from_numpy(pool).to(dev)
    pool_pin = torch.from_numpy(pool).pin_memory()
    d = torch.from_numpy(make_filters(cfg)).to(dev)
    x = torch.empty((nl, cfg.H, cfg.W), dtype=torch.float32, device=dev)
    z = torch.empty((nl, cfg.K, cfg.Hc, cfg.Wc), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    nid = cdist.broadcast_nccl_id(device=dev) if ws > 1 else None
    ctx = pkg.Context(nl, cfg.K, cfg.s, cfg.H, cfg.W, world=ws, rank=rank, device=local, stream=stream, nccl_id=nid)
    off = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.set_iter_offset(off)
    seed = mask_seed(cfg)

    def calls():
        ctx.zero_codes(x, z)
        for i in range(n_inner):
            ctx.code_step(x, d, z, cfg.lam, cfg.p, seed, i)
        ctx.filter_step(x, d, z)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    with torch.cuda.stream(stream):
        x.copy_(pool_dev[0])
        calls()
        ctx.objective(x, d, z, cfg.lam)
        torch.cuda.synchronize()
        l0 = ctx.launch_count
        ctx.objective(x, d, z, cfg.lam)
        obj_launches = ctx.launch_count - l0
        # eager steps with per-launch event timing: the kernel-class breakdown (graphs are not profiled)
        ctx.profile_enable(True)
        n_prof = 3
        for st in range(1, 1 + n_prof):
            x.copy_(pool_dev[st])
            off.fill_(n_inner * st)
            calls()
            ctx.objective(x, d, z, cfg.lam)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        torch.cuda.synchronize()
        l0 = ctx.launch_count
        graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        calls()
    graph_launches = ctx.launch_count - l0
    torch.cuda.synchronize()

    def step(st, src):
        x.copy_(src[st], non_blocking=True)
        off.fill_(n_inner * st)
        graph.replay()
        return ctx.objective(x, d, z, cfg.lam)

    with torch.cuda.stream(stream):
        st = 0
        for _ in range(args.warmup):
            step(st, pool_dev)
            st += 1
        clocks = ClockSampler(local)
        clocks.start()
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        t_total = 0.0
        objs = []
        for _ in range(args.steps):
            ev0.record(stream)
            F = step(st, pool_dev)
            ev1.record(stream)
            ev1.synchronize()
            t_total += ev0.elapsed_time(ev1)
            objs.append(F[0])
            st += 1
        torch.cuda.synchronize()
        barrier()
        clk = clocks.stop()
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        value = args.steps / (t_ms / 1e3)
        # e2e: each step's mini-batch uploaded from pinned host memory, the objective read back
        step(st, pool_pin)
        st += 1
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step(st, pool_pin)
            st += 1
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / (float(te.item()) / 1e3)
    if rank == 0:
        rl = kernel_rooflines(prof, cfg, nl, n_prof, ctx.variants)
        dom = max(rl, key=lambda k: rl[k]["ms_per_step"])
        eager_ms = sum(v[0] for v in prof.values()) / n_prof
        kernels = {k: {"ms_per_step": v[0] / n_prof, "launches_per_step": v[1] / n_prof} for k, v in prof.items()}
        line = {
            "metric": "csc_iterations_per_s", "value": value, "unit": "it/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 state; fp16 3-term split products on the tensor cores, fp32 accumulate, fp64 reductions",
            "data": "synthetic",
            "config": dict(_config_dict(cfg, ws), step="SOCSC (Alg.2): z = 0, 10 masked code steps (mask t = 10 s + i), "
                                                       "projected-gradient filter step, objective over the batch",
                           n_inner=n_inner, mini_batch=nb, cuda_graph=True,
                           l2="codes 155 MB per mini-batch (partly L2-resident); a fresh batch every step"),
            "roofline": dict(rl[dom], dominant_class=dom, note="kernel times from 3 eager profiled steps"),
            "kernel_rooflines": rl,
            "kernels": kernels,
            "eager_ms_per_step_kernels": eager_ms,
            "objective_last": objs[-1] if objs else None,
            "e2e": {"value": e2e_value, "unit": "it/s", "h2d_bytes_per_step": 4 * nl * cfg.H * cfg.W,
                    "d2h_bytes_per_step": 80},
            "gpu_launches": (graph_launches + obj_launches) * args.steps,
            "launches_per_step": graph_launches + obj_launches,
            "clocks": clk,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = _cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="sweep")
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-images", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager csc_iterate calls instead of graph replays")
    ap.add_argument("--filter-solver", default="pg", choices=["pg", "bcd", "surrogate"],
                    help="pg: the north_star projected-gradient filter step (default); bcd: the paper's "
                         "projected block-coordinate update, one warm-started sweep (SURVEY.md §8f NEXT-3); "
                         "surrogate: Eq.7 surrogate update + Eq.8 sweep per step (NEXT-2)")
    ap.add_argument("--mask", default="entry", choices=["entry", "sector8"],
                    help="entry: per-code Bernoulli (Eq.2, default); sector8: one draw per 8-code sector "
                         "(SURVEY.md §8f NEXT-4 (ii), a labelled deviation)")
    ap.add_argument("--step-rule", default="lipschitz", choices=["lipschitz", "eso"],
                    help="built-in tau_z rule of the prox code step (eso: SURVEY.md §8f NEXT-4 (i))")
    ap.add_argument("--code-solver", default="prox", choices=["prox", "admm"],
                    help="prox: the north_star masked prox-gradient step (default); admm: the paper's ADMM "
                         "code update (SURVEY.md §8f NEXT-1), 10 x 5 CG iterations")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "online" and args.code_solver == "prox" and args.filter_solver == "pg":
        run_online(args)  # the SOCSC step; the NEXT-row solvers run the iteration of run_ours on config 4
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

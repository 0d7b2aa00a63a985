"""Copy one `scripts/gpu_round2.sh TAG` record from gpurun_out/ into profiles/ (runs here, no GPU).

    python scripts/collect_round2.py TAG

Writes profiles/TAG_configs/bench_*.json (the JSON line of every bench run), TAG_pytest_gpu.log, TAG_smoke.log,
TAG_host.txt, TAG_launches.txt, TAG_trace_sweep.csv, TAG_ncu_{code_h,conv_h,wgrad_h}.txt (scripts/ncu_summary.py +
scripts/ncu_stalls.py) and refreshes profiles/traffic.json (scripts/ncu_traffic.py).
"""
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", tag)
    prof = os.path.join(ROOT, "profiles")
    cfg = os.path.join(prof, f"{tag}_configs")
    os.makedirs(cfg, exist_ok=True)
    for log in sorted(glob.glob(os.path.join(src, "bench_*.log"))):
        line = None
        for ln in open(log, errors="replace"):
            if ln.startswith("{"):
                line = ln
        name = os.path.basename(log)[:-4]
        if line is None:
            print("no JSON line in", log)
            continue
        json.dump(json.loads(line), open(os.path.join(cfg, name + ".json"), "w"), indent=1)
    for a, b in [("pytest_gpu.log", "pytest_gpu.log"), ("smoke.log", "smoke.log"), ("host.txt", "host.txt"),
                 ("launches.txt", "launches.txt"), ("trace_sweep.csv", "trace_sweep.csv")]:
        p = os.path.join(src, a)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(prof, f"{tag}_{b}"))
        else:
            print("missing", p)
    traffic = []
    for k, cls in [("code_h", "code_step"), ("conv_h", "conv"), ("wgrad_h", "wgrad")]:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{k}.ncu-rep")
        if not os.path.exists(rep):
            print("missing", rep)
            continue
        out = os.path.join(prof, f"{tag}_ncu_{k}.txt")
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), "rep", rep],
                             capture_output=True, text=True).stdout
        txt += subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_stalls.py"), rep],
                              capture_output=True, text=True).stdout
        open(out, "w").write(txt)
        traffic.append(f"{cls}={out}")
    if traffic:
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_traffic.py"), "sweep"] + traffic,
                       stdout=subprocess.DEVNULL)


if __name__ == "__main__":
    main()

"""Summarise ncu reports / launch lists into profiles/ (runs here, no GPU needed).

    python scripts/ncu_summary.py rep <file.ncu-rep> [out.txt]
    python scripts/ncu_summary.py launches <launches.csv> [out.txt]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    extra = [h for h in hdr if ("pipe_tensor_cycles_active.avg" in h or "pipe_tensor_cycles_active_realtime" in h
                                or "utchmma_src_tf32_dst_fp32_sparsity_off.avg" in h or "inst_executed_pipe_tmem.avg" in h)
             and h not in KEYS]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"kernel: {name}")
        for k in KEYS + extra:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k} = {vals[i]} {units[i]}")
    return "\n".join(out)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    unit = "?"
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("void ", "")
        name = name.split("(")[0].split("::")[-1]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        if ui is not None:
            unit = r[ui]
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)",
             f"{'kernel':40s} {'launches':>8s} {'total':>14s} {'avg':>12s} {'share':>7s}   unit={unit}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{k:40s} {cnt[k]:8d} {tot[k]:14.1f} {tot[k] / cnt[k]:12.1f} {tot[k] / allt:7.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    txt = rep(path) if mode == "rep" else launches(path)
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            f.write(txt + "\n")
    print(txt)

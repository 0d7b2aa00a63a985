"""Per-opcode and top-instruction summary of an ncu report's SASS source page (runs here, no GPU).

    python scripts/ncu_sass.py <file.ncu-rep> [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    S, E = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    by_op = defaultdict(lambda: [0, 0])
    recs = []
    tot_s = tot_e = 0
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        s, e = int(float(r[S] or 0)), int(float(r[E] or 0))
        by_op[op][0] += s
        by_op[op][1] += e
        tot_s += s
        tot_e += e
        recs.append((s, e, r[ix["Address"]][-5:], src))
    print(f"total samples {tot_s}, warp instructions executed {tot_e}")
    print(f"{'opcode':14s} {'samples':>9s} {'%':>6s} {'executed':>12s} {'%':>6s}")
    for op, (s, e) in sorted(by_op.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{op:14s} {s:9d} {100*s/max(tot_s,1):6.1f} {e:12d} {100*e/max(tot_e,1):6.1f}")
    print("\ntop instructions by stall samples:")
    for s, e, a, src in sorted(recs, key=lambda t: -t[0])[:top]:
        print(f"{s:7d} {e:10d}  {a}  {src[:90]}")


if __name__ == "__main__":
    main()

"""Stall-reason breakdown of an ncu report's SASS page, for instructions whose execution count is
in a given set (e.g. one role's per-tile body).   python scripts/ncu_stalls.py <rep> [exec_count ...]"""
import csv
import io
import subprocess
import sys
from collections import Counter

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(raw.splitlines()[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
want = set(int(x) for x in sys.argv[2:])
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
per_op = Counter()
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    e = int(float(r[ix["Instructions Executed"]] or 0))
    if want and e not in want:
        continue
    for h in reasons:
        v = float(r[ix[h]] or 0)
        tot[h] += v
    op = r[ix["Source"]].split()
    op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    per_op[op.split(".")[0]] += sum(float(r[ix[h]] or 0) for h in reasons)
s = sum(tot.values())
for h, v in tot.most_common(12):
    print(f"{h:24s} {v:9.0f} {100 * v / max(s, 1):5.1f}%")
print("by opcode:", per_op.most_common(10))

"""Collect per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels
captured with `ncu --set full` (summaries profiles/<tag>_ncu_<kernel>.txt written by
scripts/ncu_summary.py) into profiles/traffic.json, keyed by bench kernel class and config.

    python scripts/ncu_traffic.py <config> <class>=<summary.txt> [...]
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    cfg = sys.argv[1]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for arg in sys.argv[2:]:
        cls, path = arg.split("=", 1)
        tot = 0.0
        for line in open(path):
            m = re.match(r"\s*dram__bytes_(read|write)\.sum = ([0-9.]+) (\w+)", line)
            if m:
                tot += float(m.group(2)) * UNITS[m.group(3)]
        data.setdefault(cls, {})[cfg] = {"bytes_per_launch": tot, "source": os.path.relpath(path, ROOT)}
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()

"""Summarise tools/bench_rt.py output files: runtime-kernel fraction of HBM peak per config / pattern."""
import json
import sys

for fn in sys.argv[1:]:
    cells = []
    for line in open(fn):
        d = json.loads(line)
        if d.get("kernel") == "ring_rt" and "cfg" in d:
            cells.append(f"c{d['cfg']}={d['frac']:.3f}")
        elif d.get("kernel") == "ring_rt" and "code" in d:
            cells.append(f"{d['code']} {d['op']}={d['frac']:.3f}")
        elif "pattern" in d:
            cells.append(f"{''.join(map(str, d['pattern']))}={d['frac']:.3f}")
    print(fn.split("/")[-1], " ".join(cells))

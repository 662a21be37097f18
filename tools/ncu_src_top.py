"""Top stall sites of an `ncu --page source --csv --print-source sass` dump.

    python tools/ncu_src_top.py src.csv [N]

Prints the N SASS instructions with most warp-stall samples (with the dominant
stall reasons of each) and the per-opcode totals.
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) >= len(hdr) - 2 and r[0].startswith("0x") or (hdr and r and r[0].isdigit()):
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


total = sum(num(r[ix["# Samples"]]) for r in data)
print("instructions", len(data), "samples", total)
tot = defaultdict(float)
for r in data:
    for s in stalls:
        tot[s] += num(r[ix[s]])
print("by reason:", ", ".join(f"{s[6:]} {v / total:.3f}" for s, v in sorted(tot.items(), key=lambda t: -t[1]) if v))
byop = defaultdict(lambda: [0.0, 0.0])
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    byop[op][0] += num(r[ix["# Samples"]])
    byop[op][1] += num(r[ix["Instructions Executed"]])
print("by opcode (samples share, executed):")
for op, (s, e) in sorted(byop.items(), key=lambda t: -t[1][0])[:14]:
    print(f"  {op:14s} {s / total:.3f} {int(e)}")
print("top sites:")
for r in sorted(data, key=lambda r: -num(r[ix["# Samples"]]))[:top]:
    why = sorted(((num(r[ix[s]]), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"  {r[0]:>8s} {num(r[ix['# Samples']]) / total:.4f} exec {int(num(r[ix['Instructions Executed']])):>9d} "
          f"{r[ix['Source']][:52]:52s} " + " ".join(f"{n}:{int(v)}" for v, n in why if v))

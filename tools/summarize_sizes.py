#!/usr/bin/env python
"""Markdown table from tools/bench_sizes.py JSON lines."""
import json
import sys

for fn in sys.argv[1:]:
    rows = [json.loads(l) for l in open(fn) if l.startswith("{")]
    if not rows:
        continue
    d0 = rows[0]
    print(f"\n{fn}: k={d0['k']} r={d0['r']} {d0['field']} transform={d0['transform']}\n")
    print("| size | op | codec | stripes/launch | GPU src GB/s | GPU moved GB/s | ref CPU src GB/s | GPU/CPU | kernel |")
    print("|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        cpu = d.get("cpu_src_GBps")
        print(f"| {d['size']} | {d['op']} | {d['codec']} | {d['stripes']} | {d['gpu_src_GBps']:.0f} | "
              f"{d['gpu_moved_GBps']:.0f} | {cpu:.2f} | {d['gpu_src_GBps'] / cpu:.0f}x | " if cpu else
              f"| {d['size']} | {d['op']} | {d['codec']} | {d['stripes']} | {d['gpu_src_GBps']:.0f} | "
              f"{d['gpu_moved_GBps']:.0f} | - | - | ", end="")
        print(d["kernel"].split("_")[-2] + " |")

#!/usr/bin/env python
"""H2D bandwidth from pinned memory with 1, 2 and 4 concurrent streams (same total bytes):
does splitting the host->device copies over several streams / copy engines beat one?"""
import json
import time

import torch

dev = torch.device("cuda", 0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=dev)
res = {}
for ns in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    d[:part].copy_(h[:part], non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(4):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    bw = 4 * n / (time.perf_counter() - t) / 1e9
    res.setdefault(f"h2d_{ns}_streams_GBps", []).append(round(bw, 2))
print(json.dumps(res))

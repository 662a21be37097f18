#!/usr/bin/env python
"""Host<->device copy bandwidth on this box (context for the e2e number)."""
import json
import time

import torch

dev = torch.device("cuda", 0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n // 4, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n // 4, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    res[name + "_GBps"] = 5 * n / (time.perf_counter() - t) / 1e9
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
el = time.perf_counter() - t
res["bidir_h2d_1GiB_plus_d2h_256MiB_GBps_h2d_side"] = 5 * n / el / 1e9
print(json.dumps(res))

#!/usr/bin/env python
"""Sustained device copy (torch) with clock/power sampling: the power reference for bench numbers."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402

n = 5 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 150
with ClockSampler(0) as clk:
    e0.record()
    for _ in range(steps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(json.dumps({"copy_GBps": 2 * n / ms / 1e6, "ms": ms, "clocks": clk.summary()}))

#!/usr/bin/env python
"""Tiny launches of the runtime-matrix kernel (config-5 shape, 4 erasures, 12 x 4 KiB
strips): host microseconds per enqueue and device microseconds per launch."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200 import _lib as L  # noqa: E402

lib = L.load()
L.check(lib.pyrit_set_kernel_mode(4))
code = P.CodeSpec(16, 4, P.FieldSpec.aop(12))
dev = torch.device("cuda", 0)
out = {}
for strips_kib in (4, 64, 1024):
    strip = strips_kib * 1024
    ss = 12 * strip
    sym = torch.zeros((20, ss), dtype=torch.uint8, device=dev)
    plan = P.Plan.decode(code, (0, 5, 16, 19))
    ins = (C.c_void_p * 16)(*[sym[s].data_ptr() for s in plan.survivors])
    outs = (C.c_void_p * 4)(*[sym[o].data_ptr() for o in plan.outputs])
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(20):
        lib.pyrit_cu_apply(plan._h, ins, outs, strip, 0, strip, st)
    torch.cuda.synchronize()
    kern = P.Plan.last_launch()["kernel"]
    host, devus = [], []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0.record()
        for _ in range(32):
            lib.pyrit_cu_apply(plan._h, ins, outs, strip, 0, strip, st)
        e1.record()
        host.append((time.perf_counter() - t) / 32 * 1e6)
        torch.cuda.synchronize()
        devus.append(e0.elapsed_time(e1) * 1000 / 32)
    host.sort(), devus.sort()
    out[f"strip_{strips_kib}KiB"] = {"kernel": kern, "host_us": round(host[10], 2), "device_us": round(devus[10], 2)}
print(json.dumps(out))

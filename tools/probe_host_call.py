#!/usr/bin/env python
"""Fixed host cost of one pyrit_encode_host call: tiny symbols (config-1 code, 16-byte strips)
through the Python wrapper and straight through ctypes, median of 200 calls."""
import ctypes as C
import json
import os
import sys
import time

os.environ.setdefault("PYRIT_B200_TIERED", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200 import _lib as L  # noqa: E402
from paper_1709_00178_b200.workloads import WORKLOADS  # noqa: E402

lib = L.load()
wl = WORKLOADS[1]
for strip in (16, 4096, 65536, wl.strip):
    sym = wl.fld.w * strip
    hin = torch.zeros((wl.k, sym), dtype=torch.uint8, pin_memory=True)
    hout = torch.zeros((wl.m, sym), dtype=torch.uint8, pin_memory=True)
    a_in, a_out = hin.numpy(), hout.numpy()
    code = wl.code.c()
    res = {"strip": strip, "bytes_in": wl.k * sym}
    for label, fn in (("python", lambda: P.encode_host(a_in, wl.code, device=0, parity=a_out)),
                      ("ctypes", lambda: L.check(lib.pyrit_encode_host(C.byref(code), a_in.ctypes.data, a_out.ctypes.data, sym, 0)))):
        for _ in range(10):
            fn()
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        res[label + "_us"] = round(ts[len(ts) // 2] * 1e6, 1)
    print(json.dumps(res), flush=True)

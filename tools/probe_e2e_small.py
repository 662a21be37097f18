#!/usr/bin/env python
"""Host-buffer encode of the small BASELINE configs (1, 2) through pyrit_encode_host: median
wall time per call for several staging chunk sizes (pyrit_set_host_chunk; 0 = the default rule).

    python tools/probe_e2e_small.py
"""
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
for c in (1, 2):
    wl = WORKLOADS[c]
    sym = wl.frag
    hin = torch.empty((wl.k, sym), dtype=torch.uint8, pin_memory=True)
    hout = torch.empty((wl.m, sym), dtype=torch.uint8, pin_memory=True)
    a_in, a_out = hin.numpy(), hout.numpy()
    a_in[...] = np.random.default_rng(0).integers(0, 256, a_in.shape, dtype=np.uint8)
    for ch in (0, wl.strip, wl.strip // 2, wl.strip // 4, wl.strip // 8):
        L.check(lib.pyrit_set_host_chunk(ch))
        for _ in range(5):
            P.encode_host(a_in, wl.code, device=0, parity=a_out)
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            P.encode_host(a_in, wl.code, device=0, parity=a_out)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        med = ts[len(ts) // 2]
        print(json.dumps({"cfg": c, "chunk": ch, "chunks": (-(-wl.strip // ch) if ch else "default"),
                          "median_ms": round(med * 1e3, 3), "src_GBps": round(wl.k * sym / med / 1e9, 1)}), flush=True)
    L.check(lib.pyrit_set_host_chunk(0))

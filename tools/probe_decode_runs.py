#!/usr/bin/env python
"""Host-buffer decode (pinned) of config 4 with different erasure patterns: survivors/outputs in
one contiguous run vs scattered runs (one 2D copy per run and chunk).
    python tools/probe_decode_runs.py"""
from __future__ import annotations

import json
import os
import sys
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200.workloads import WORKLOADS
    wl = WORKLOADS[4]
    host = torch.empty((wl.k + wl.m, wl.frag), dtype=torch.uint8).pin_memory()
    host.numpy()[:] = np.random.default_rng(0).integers(0, 256, (wl.k + wl.m, wl.frag), dtype=np.uint8)
    a = host.numpy()
    for erased in ([10, 11, 12, 13], [1, 6, 9, 10], [0, 1, 2, 3], [1, 3, 5, 7]):
        P.decode_host(a, erased, wl.code)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            P.decode_host(a, erased, wl.code)
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(json.dumps({"erased": erased, "ms": t * 1e3, "src_GBps": wl.k * wl.frag / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Host-buffer encode/decode from pageable vs pinned memory (the shim's SymbolBuffer is a
std::vector: pageable).  python tools/probe_pageable.py [--config 3] [--reps 3]"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200.workloads import WORKLOADS

    wl = WORKLOADS[a.config]
    rng = np.random.default_rng(0)
    data_pg = rng.integers(0, 256, (wl.k, wl.frag), dtype=np.uint8)
    par_pg = np.empty((wl.m, wl.frag), dtype=np.uint8)
    data_pin = torch.empty((wl.k, wl.frag), dtype=torch.uint8).pin_memory()
    data_pin.numpy()[:] = data_pg
    par_pin = torch.empty((wl.m, wl.frag), dtype=torch.uint8).pin_memory()
    for name, d, p in (("pageable", data_pg, par_pg), ("pinned", data_pin.numpy(), par_pin.numpy())):
        P.encode_host(d, wl.code, parity=p)  # warm-up (plan, kernel, staging)
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            P.encode_host(d, wl.code, parity=p)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(json.dumps({"workload": wl.name, "memory": name, "s": t, "src_GBps": wl.k * wl.frag / t / 1e9,
                          "h2d_bytes": wl.k * wl.frag, "d2h_bytes": wl.m * wl.frag}), flush=True)
    assert np.array_equal(par_pg, par_pin.numpy())


if __name__ == "__main__" and not os.environ.get("PROBE_REGISTER"):
    main()


def probe_register():
    """cudaHostRegister / cudaHostUnregister cost on a touched pageable buffer (GB/s of pages)."""
    import numpy as np
    import torch
    cr = torch.cuda.cudart()
    torch.cuda.init()
    for gib in (1, 4):
        buf = np.ones(gib << 30, dtype=np.uint8)
        t0 = time.perf_counter()
        rc = cr.cudaHostRegister(buf.ctypes.data, buf.nbytes, 0)
        t1 = time.perf_counter()
        rc2 = cr.cudaHostUnregister(buf.ctypes.data)
        t2 = time.perf_counter()
        print(json.dumps({"register_GiB": gib, "rc": int(rc), "register_s": t1 - t0, "unregister_s": t2 - t1,
                          "register_GBps": buf.nbytes / (t1 - t0) / 1e9, "rc2": int(rc2)}), flush=True)


if __name__ == "__main__" and os.environ.get("PROBE_REGISTER"):
    probe_register()

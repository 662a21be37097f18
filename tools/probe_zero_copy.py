#!/usr/bin/env python
"""Zero-copy experiment: the fused kernel reading its inputs straight from pinned host memory and
writing its outputs there (UVA pointers, no staging copies), vs the staged host pipeline.
    python tools/probe_zero_copy.py"""
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
    from paper_1709_00178_b200 import _lib as L
    from paper_1709_00178_b200.workloads import WORKLOADS
    lib = L.load()
    for cfg in (3, 5):
        wl = WORKLOADS[cfg]
        w = wl.fld.w
        data = torch.empty((wl.k, wl.frag), dtype=torch.uint8).pin_memory()
        data.numpy()[:] = np.random.default_rng(0).integers(0, 256, (wl.k, wl.frag), dtype=np.uint8)
        par = torch.empty((wl.m, wl.frag), dtype=torch.uint8).pin_memory()
        plan = P.Plan.encode(wl.code)
        ins = [data[j].data_ptr() for j in range(wl.k)]
        outs = [par[i].data_ptr() for i in range(wl.m)]
        st = torch.cuda.current_stream().cuda_stream
        for mode in (1, 2):
            L.check(lib.pyrit_set_kernel_mode(mode))
            try:
                plan.apply(ins, outs, wl.strip, stream=st)
                torch.cuda.synchronize()
                ts = []
                for _ in range(3):
                    t0 = time.perf_counter()
                    plan.apply(ins, outs, wl.strip, stream=st)
                    torch.cuda.synchronize()
                    ts.append(time.perf_counter() - t0)
                t = min(ts)
                ref = P.encode_host(data.numpy(), wl.code)
                print(json.dumps({"workload": wl.name, "mode": mode, "kernel": P.Plan.last_launch()["kernel"],
                                  "s": t, "src_GBps": wl.k * wl.frag / t / 1e9,
                                  "correct": bool(np.array_equal(ref, par.numpy()))}), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"workload": wl.name, "mode": mode, "error": str(e)[:300]}), flush=True)
        L.check(lib.pyrit_set_kernel_mode(0))
        t0 = time.perf_counter()
        P.encode_host(data.numpy(), wl.code, parity=par.numpy())
        t = time.perf_counter() - t0
        print(json.dumps({"workload": wl.name, "mode": "staged pipeline", "src_GBps": wl.k * wl.frag / t / 1e9}))
        del data, par


if __name__ == "__main__":
    main()

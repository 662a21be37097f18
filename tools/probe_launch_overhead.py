#!/usr/bin/env python
"""Host cost of one C-ABI launch (no CUDA graph): wall time per pyrit_cu_apply / pyrit_cu_encode call
on small device buffers, against the same launches captured in a graph.
    python tools/probe_launch_overhead.py"""
from __future__ import annotations

import json
import os
import sys
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200.workloads import WORKLOADS
    dev = torch.device("cuda", 0)
    for cfg, strip in ((1, 4096), (5, 4096), (5, 16 * 65536)):
        wl = WORKLOADS[cfg]
        w = wl.fld.w
        data = torch.randint(0, 256, (wl.k, w * strip), dtype=torch.uint8, device=dev)
        par = torch.empty((wl.m, w * strip), dtype=torch.uint8, device=dev)
        plan = P.Plan.encode(wl.code)
        ins = [data[j].data_ptr() for j in range(wl.k)]
        outs = [par[i].data_ptr() for i in range(wl.m)]
        st = torch.cuda.current_stream(dev).cuda_stream
        for _ in range(20):
            plan.apply(ins, outs, strip, stream=st)
        torch.cuda.synchronize()
        n = 2000
        t0 = time.perf_counter()
        for _ in range(n):
            plan.apply(ins, outs, strip, stream=st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream().cuda_stream
            for _ in range(100):
                plan.apply(ins, outs, strip, stream=cs)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"workload": wl.name, "strip": strip, "kernel": P.Plan.last_launch()["kernel"],
                          "host_us_per_call": (t1 - t0) / n * 1e6, "wall_us_per_call": (t2 - t0) / n * 1e6,
                          "graph_us_per_launch": e0.elapsed_time(e1) * 1000 / 100}), flush=True)


if __name__ == "__main__":
    main()

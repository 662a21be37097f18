#!/usr/bin/env python
"""Each BASELINE config's kernel against a plain device copy of the same bytes.

    python tools/copy_floor.py [--configs 1,2,3,4,5] [--steps 50]

For every config: the bench's step (the specialised kernel over buffer sets
rotated until the working set exceeds 4x L2) and torch's device-to-device copy
moving the same number of bytes ((k+m)·F or (k+e)·F: half read, half written),
both as CUDA graphs of `steps` launches, best of 5 replays.  `kernel_vs_copy`
= copy time / kernel time: 1.0 means the kernel costs exactly what moving its
bytes costs at this size (launch, ramp and DRAM latency included).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

os.environ.setdefault("PYRIT_B200_TIERED", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200.workloads import WORKLOADS  # noqa: E402


def graph_ms(fn, steps):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(steps):
            fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps
        best = t if best is None else min(best, t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for c in [int(x) for x in a.configs.split(",")]:
        wl = WORKLOADS[c]
        nout = wl.m if wl.op == "encode" else len(wl.erased)
        moved = (wl.k + nout) * wl.frag
        nsets = max(1, -(-4 * l2 // moved))
        steps = max(a.steps if moved < (1 << 30) else 10, nsets)
        sets = []
        for _ in range(nsets):
            buf = torch.empty((wl.k + wl.m, wl.frag), dtype=torch.uint8, device=dev)
            for j in range(wl.k):
                P.fill(buf[j], wl.seed, j, valid=wl.valid)
            sets.append(buf)
        if wl.op == "encode":
            plan = P.Plan.encode(wl.code)
            ptrs = [([b[j].data_ptr() for j in range(wl.k)], [b[wl.k + i].data_ptr() for i in range(wl.m)])
                    for b in sets]
        else:
            enc = P.Plan.encode(wl.code)
            for b in sets:
                enc.apply([b[j].data_ptr() for j in range(wl.k)], [b[wl.k + i].data_ptr() for i in range(wl.m)],
                          wl.strip)
            plan = P.Plan.decode(wl.code, wl.erased)
            ptrs = [([b[s].data_ptr() for s in plan.survivors], [b[o].data_ptr() for o in plan.outputs]) for b in sets]
        torch.cuda.synchronize()

        def step(i):
            ins, outs = ptrs[i % nsets]
            plan.apply(ins, outs, wl.strip, stream=torch.cuda.current_stream().cuda_stream)

        step(0)
        torch.cuda.synchronize()
        kern = P.Plan.last_launch()["kernel"]
        k_ms = graph_ms(step, steps)
        half = moved // 2
        srcs = [s.view(-1)[:half] for s in sets]
        dsts = [torch.empty(half, dtype=torch.uint8, device=dev) for _ in range(nsets)]
        c_ms = graph_ms(lambda i: dsts[i % nsets].copy_(srcs[i % nsets]), steps)
        print(json.dumps({"cfg": c, "kernel": kern, "moved_bytes": moved, "rotating_sets": nsets, "steps": steps,
                          "kernel_us": round(k_ms * 1e3, 2), "copy_us": round(c_ms * 1e3, 2),
                          "kernel_vs_copy": round(c_ms / k_ms, 3),
                          "kernel_moved_GBps": round(moved / k_ms / 1e6, 1),
                          "copy_moved_GBps": round(moved / c_ms / 1e6, 1)}), flush=True)
        del sets, dsts, srcs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

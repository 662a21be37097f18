#!/usr/bin/env python
"""Config 1 (6 MiB per launch): separate kernel time from launch time.

    python tools/cfg1_launch.py [--steps 200]

Three CUDA graphs of `steps` launches each, replayed and timed with CUDA events:
  * cfg1  -- the bench's step (the encode kernel over rotating buffer sets > L2);
  * floor -- the same number of launches of a near-empty kernel (pyrit_cu_fill of
             8 bytes: one CTA), i.e. the graph's launch-to-launch floor;
  * floor_wide -- an 8-byte fill launched as a 148 x 256 grid: the floor for a
             grid the size of the encode kernel's.
and, for each kernel choice of config 1 (direct, staged, runtime-matrix), the
per-launch time.  ms per step - floor = what the kernel itself adds.
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
from paper_1709_00178_b200 import _lib as L  # noqa: E402
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    lib = L.load()
    dev = torch.device("cuda", 0)
    wl = WORKLOADS[1]
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    moved = (wl.k + wl.m) * wl.frag
    nsets = max(1, -(-4 * l2 // moved))
    sets = []
    for _ in range(nsets):
        d = torch.empty((wl.k, wl.frag), dtype=torch.uint8, device=dev)
        for j in range(wl.k):
            P.fill(d[j], wl.seed, j, valid=wl.valid)
        par = torch.empty((wl.m, wl.frag), dtype=torch.uint8, device=dev)
        sets.append(([d[j].data_ptr() for j in range(wl.k)], [par[i].data_ptr() for i in range(wl.m)], d, par))
    plan = P.Plan.encode(wl.code)
    res = {"config": wl.name, "bytes_moved_per_launch": moved, "rotating_sets": nsets, "steps": a.steps}
    for name, mode in (("auto", 0), ("direct", 1), ("staged", 2), ("ring_rt", 4)):
        L.check(lib.pyrit_set_kernel_mode(mode))
        try:
            def step(i):
                plan.apply(sets[i % nsets][0], sets[i % nsets][1], wl.strip,
                           stream=torch.cuda.current_stream().cuda_stream)
            step(0)
            torch.cuda.synchronize()
            k = P.Plan.last_launch()
            ms = graph_ms(step, a.steps)
            res[name] = {"us_per_launch": round(ms * 1e3, 3), "kernel": k["kernel"], "grid": [k["blocks"], k["threads"]],
                         "moved_GBps": round(moved / ms / 1e6, 1)}
        finally:
            L.check(lib.pyrit_set_kernel_mode(0))
    buf = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    res["floor_fill_8B"] = {"us_per_launch": round(graph_ms(lambda i: P.fill(buf[:8], 1, i % 7, stream=st()),
                                                            a.steps) * 1e3, 3), "grid": [1, 256]}
    wide = 148 * 256 * 8
    res["floor_fill_wide"] = {"us_per_launch": round(graph_ms(lambda i: P.fill(buf[:wide], 1, i % 7, stream=st()),
                                                              a.steps) * 1e3, 3),
                              "grid": [148, 256], "bytes": wide}
    # the same bytes through library kernels, same rotating sets and graph: torch's
    # XOR of two 2 MiB halves of each set's data (4 MiB read, 2 MiB written, like
    # config 1's 4 MiB in / 2 MiB out) and a 6 MiB device-to-device copy (3 + 3)
    half = wl.k * wl.frag // 2
    flat = [s[2].view(-1) for s in sets]
    outs = [s[3].view(-1) for s in sets]

    def xor_step(i):
        f = flat[i % nsets]
        torch.bitwise_xor(f[:half], f[half:2 * half], out=outs[i % nsets][:half])

    res["torch_xor_4MiB_in_2MiB_out"] = {"us_per_launch": round(graph_ms(xor_step, a.steps) * 1e3, 3),
                                         "bytes": 3 * half}
    cp_src = [torch.empty(moved // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
    cp_dst = [torch.empty(moved // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
    res["torch_copy_3MiB"] = {"us_per_launch": round(graph_ms(lambda i: cp_dst[i % nsets].copy_(cp_src[i % nsets]),
                                                              a.steps) * 1e3, 3), "bytes": moved}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-GPU work at 1/2/4/8-way byte-offset sharding, measured on one GPU.

    python tools/shard_scaling.py [--config 5] [--steps 20]

The hot path shards with no exchange: at N GPUs each rank runs the
same kernel on its [lo, hi) byte range of every strip.  This measures rank 0's
shard at N = 1, 2, 4, 8 on one device (CUDA graph of K launches, events, the
clock sampler started first, as bench.py) and reports the aggregate the job would
reach if every rank ran at that speed -- the upper bound of strong scaling that
launch overhead and tail effects leave.  It is a projection for the scaling
row, not a multi-GPU measurement (bench.py under torchrun is that).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--only", type=int, nargs="*", default=None, help="shard counts to run (default 1 2 4 8)")
    a = ap.parse_args()

    import torch

    import paper_1709_00178_b200 as P
    from bench import ClockSampler
    from paper_1709_00178_b200.workloads import WORKLOADS, shard

    dev = torch.device("cuda", 0)
    wl = WORKLOADS[a.config]
    w = wl.fld.w
    if wl.op == "encode":
        plan = P.Plan.encode(wl.code)
        n_in, n_out = wl.k, wl.m
    else:  # the repair program over k survivors (inputs are arbitrary bytes: timing only)
        plan = P.Plan.decode(wl.code, wl.erased)
        n_in, n_out = wl.k, len(wl.erased)
    base = None
    for n in a.only or (1, 2, 4, 8):
        lo, hi = shard(wl.strip, 0, n)
        Ls = hi - lo
        sym = w * Ls
        data = torch.empty((n_in, sym), dtype=torch.uint8, device=dev)
        for j in range(n_in):
            for s in range(w):
                P.fill(data[j, s * Ls:(s + 1) * Ls], wl.seed, j, begin=s * wl.strip + lo, valid=wl.valid)
        par = torch.empty((n_out, sym), dtype=torch.uint8, device=dev)
        ins = [data[j].data_ptr() for j in range(n_in)]
        outs = [par[i].data_ptr() for i in range(n_out)]
        st = torch.cuda.current_stream(dev).cuda_stream
        for _ in range(a.warmup):
            plan.apply(ins, outs, Ls, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream().cuda_stream
            for _ in range(a.steps):
                plan.apply(ins, outs, Ls, stream=cs)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        agg = wl.source_bytes() / (ms * 1e-3) / 1e9  # every rank at rank 0's speed
        base = base or agg
        print(json.dumps({"workload": wl.name, "n_gpus": n, "shard_strip_bytes": Ls, "ms_per_step": ms,
                          "rank_moved_GBps": (n_in + n_out) * sym / (ms * 1e-3) / 1e9,
                          "projected_aggregate_src_GBps": agg, "projected_efficiency": agg / (n * base),
                          "kernel": P.Plan.last_launch()["kernel"], "clocks": clk.summary()}), flush=True)
        del g, data, par
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

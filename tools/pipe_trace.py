#!/usr/bin/env python
"""Timeline of one host-buffer encode/decode call (pyrit_encode_host / pyrit_decode_host):
per-chunk CUDA events around H2D, kernel and D2H (PYRIT_B200_PIPE_TRACE), summarised
as copy-engine busy time and overlap -- the evidence an nsys timeline would give.

    python tools/pipe_trace.py [--config 5] [--out profiles/r02/pipe_trace_cfg5.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot


def overlap(a_iv, b_iv):
    return union(a_iv) + union(b_iv) - union(a_iv + b_iv)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    trace = tempfile.mktemp(suffix=".jsonl")
    os.environ["PYRIT_B200_PIPE_TRACE"] = trace
    import torch
    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200.workloads import WORKLOADS
    wl = WORKLOADS[a.config]
    if wl.op == "encode":
        hin = torch.empty((wl.k, wl.frag), dtype=torch.uint8, pin_memory=True)
        hout = torch.empty((wl.m, wl.frag), dtype=torch.uint8, pin_memory=True)
        hin.random_(0, 256)
        call = lambda: P.encode_host(hin.numpy(), wl.code, parity=hout.numpy())  # noqa: E731
    else:
        h = torch.empty((wl.k + wl.m, wl.frag), dtype=torch.uint8, pin_memory=True)
        h.random_(0, 256)
        call = lambda: P.decode_host(h.numpy(), wl.erased, wl.code)  # noqa: E731
    call()
    os.remove(trace) if os.path.exists(trace) else None
    t0 = time.perf_counter()
    call()
    wall = (time.perf_counter() - t0) * 1e3
    rec = json.loads(open(trace).read().splitlines()[-1])
    ch = rec["chunks"]
    h2d = [tuple(c["h2d"]) for c in ch]
    k = [tuple(c["kernel"]) for c in ch]
    d2h = [tuple(c["d2h"]) for c in ch]
    span = max(c["d2h"][1] for c in ch)
    hb = sum(c["h2d_bytes"] for c in ch)
    db = sum(c["d2h_bytes"] for c in ch)
    summ = {"config": wl.name, "wall_ms": round(wall, 2), "events_span_ms": round(span, 2), "chunks": len(ch),
            "h2d_busy_ms": round(union(h2d), 2), "d2h_busy_ms": round(union(d2h), 2),
            "kernel_busy_ms": round(union(k), 2), "h2d_d2h_overlap_ms": round(overlap(h2d, d2h), 2),
            "h2d_GBps_while_busy": round(hb / union(h2d) / 1e6, 1), "d2h_GBps_while_busy": round(db / union(d2h) / 1e6, 1),
            "source_GBps_wall": round(wl.source_bytes() / wall / 1e6, 1), "h2d_bytes": hb, "d2h_bytes": db,
            "note": "event intervals are stream-ordered: an H2D interval opens when its stream reaches it, so "
                    "busy time is an upper bound of the copy engine's own time"}
    print(json.dumps(summ))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summ, "chunks": ch}, f)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Symbol-size sweep: the reference's `pyrit bench` (bench.hpp:54-58 sizes
128 B .. 8 MiB, codecs pyrit / crs, ops encode / decode) on the GPU, with
stripe batching (one launch covers every stripe of a > L2 working set).

    python tools/bench_sizes.py --k 8 --r 4 --field gf16 [--transform 0] \
        [--sizes 128,...] [--codec pyrit,crs] [--op encode,decode] [--cpu]

GPU point: nb stripes of `size`-byte symbols, device resident (encode: the
input-file layout, stripe = k symbols, parity written in shard order;
decode: shard-major symbols, erased data {0..min(k,r)-1} as BenchRunner,
bench.hpp:124-134).  K launches captured in a CUDA graph, CUDA events.
Rates: source GB/s (k * size per stripe) and the reference's (k+r) * size
convention (bench.hpp:205-207).  --cpu adds the reference itself (oracle/_ref):
its own bench cell BenchRunner::run_point (bench.hpp:146-208, one stripe,
column windows over 1 and all host threads, best of the two) for w <= 6, else a
precompiled schedule + parallel_replay on one stripe.  One JSON line per point.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FIELDS = {"gf16": (4, 5, 0, 1, 4, 0x1F), "gf64": (6, 9, 1, 3, 2, 0x49), "gf256_r17": (8, 17, 0, 1, 8, 0x139),
          "gf1024": (10, 11, 0, 1, 10, 0x7FF), "gf4096": (12, 13, 0, 1, 12, 0x1FFF)}


def cpu_point(f, k, r, kind, size, op, codec, threads, seconds=0.25):
    """Seconds per stripe of the reference CPU path.  Fields with w <= 6: the
    reference's own bench cell (BenchRunner::run_point, bench.hpp:146-208), best
    of 1 and `threads` workers; wider fields (BenchRunner cannot build its table
    codec there): precompiled schedule + parallel_replay with `threads`."""
    import numpy as np

    import oracle as O
    of = O.Field(*f)
    if f[0] <= 6:
        best = 0.0
        for t in sorted({1, threads}):
            g = O.ref_bench_point(of, k, r, 1 if codec == "crs" else 0, 0 if op == "encode" else 1, size, t, kind,
                                  seconds)
            best = max(best, g)
        return (k + r) * size / (best * 1e9) if best > 0 else None
    if op == "encode":
        mode = 1 if codec == "crs" else 0
        erased = ()
    else:
        mode = 2 if codec == "crs" else 3
        erased = tuple(range(min(k, r)))
    if kind:
        if codec == "crs":
            return None
        mode |= 0x10
    if f[1] > 16 and codec != "crs":
        return None  # the reference's ring path is wrong for R_{2,17}
    plan = O.RefPlan(of, k, r, mode, size, erased)
    rng = np.random.default_rng(size)
    for s in range(k + r):
        plan.symbol(s)[:] = rng.integers(0, 256, size, dtype=np.uint8)
    plan.run(threads)
    iters, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or iters < 3:
        plan.run(threads)
        iters += 1
    dt = (time.perf_counter() - t0) / iters
    plan.close()
    return dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--r", type=int, default=4)
    ap.add_argument("--field", default="gf16", choices=sorted(FIELDS))
    ap.add_argument("--transform", type=int, default=0)
    ap.add_argument("--sizes", default="")
    ap.add_argument("--codec", default="pyrit,crs")
    ap.add_argument("--op", default="encode,decode")
    ap.add_argument("--bytes", type=int, default=1 << 30, help="source bytes per launch (working set > L2)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--mode", type=int, default=0, help="kernel mode: 0 auto, 1 direct, 2 staged")
    a = ap.parse_args()

    import torch

    import paper_1709_00178_b200 as P

    from paper_1709_00178_b200 import _lib as L
    L.check(L.load().pyrit_set_kernel_mode(a.mode))
    dev = torch.device("cuda", 0)
    f = FIELDS[a.field]
    fs = P.FieldSpec(*f)
    k, r = a.k, a.r
    code = P.CodeSpec(k, r, fs, P.TransformKind(a.transform))
    unit = f[0] * 8 // math.gcd(f[0], 8)  # lcm(w, 8): pyrit.cpp:35-38 round_symbol_size
    sizes = [int(s) for s in a.sizes.split(",")] if a.sizes else [128 << i for i in range(17)]
    threads = os.cpu_count() or 1
    stream = torch.cuda.current_stream(dev).cuda_stream
    for req in sizes:
        size = (req + unit - 1) // unit * unit
        nb = max(1, a.bytes // (k * size))
        strip = size // f[0]
        for op in a.op.split(","):
            for codec in a.codec.split(","):
                if codec == "crs" and a.transform:
                    continue
                rep = P.RingRep.Crs if codec == "crs" else P.RingRep.Sparse
                m = P.cauchy_parity_matrix(code)
                if op == "encode":
                    plan = P.Plan.create(fs, m, P.TransformKind(a.transform), rep)
                    data = torch.empty((nb, k * size), dtype=torch.uint8, device=dev)
                    P.fill(data.view(-1), 7, 0)
                    out = torch.empty((r, nb, size), dtype=torch.uint8, device=dev)
                    ins = [data.data_ptr() + j * size for j in range(k)]
                    outs = [out[i].data_ptr() for i in range(r)]
                    in_pitch, out_pitch, n_out = k * size, size, r
                else:
                    erased = list(range(min(k, r)))
                    surv, order, dm = P.repair_matrix(code, erased)
                    plan = P.Plan.create(fs, dm, P.TransformKind(a.transform), rep)
                    sym = torch.empty((k + r, nb, size), dtype=torch.uint8, device=dev)
                    P.fill(sym.view(-1), 8, 0)
                    ins = [sym[s].data_ptr() for s in surv]
                    outs = [sym[o].data_ptr() for o in order]
                    in_pitch = out_pitch = size
                    n_out = len(order)

                def launch(s=stream):
                    plan.apply_batch(ins, outs, strip, nb, in_pitch, out_pitch, stream=s)

                for _ in range(a.warmup):
                    launch()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    cs = torch.cuda.current_stream().cuda_stream
                    for _ in range(a.steps):
                        launch(cs)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.steps
                info = P.Plan.last_launch()
                src = k * size * nb
                row = {"mode": a.mode, "field": a.field, "k": k, "r": r, "transform": a.transform, "op": op, "codec": codec,
                       "size": size, "stripes": nb, "gpu_ms": ms, "gpu_src_GBps": src / ms / 1e6,
                       "gpu_ref_GBps": (k + r) * size * nb / ms / 1e6,
                       "gpu_moved_GBps": (k + n_out) * size * nb / ms / 1e6, "kernel": info["kernel"],
                       "xors_per_word": plan.stats()["part_xors" if ("_cpa" in info["kernel"] or "_tm" in
                                                                     info["kernel"]) else "xors"]}
                if a.cpu:
                    dt = cpu_point(f, k, r, a.transform, size, op, codec, threads)
                    if dt:
                        row.update({"cpu_threads": threads, "cpu_src_GBps": k * size / dt / 1e9,
                                    "cpu_ref_GBps": (k + r) * size / dt / 1e9})
                print(json.dumps(row), flush=True)
                del g
                plan.close()


if __name__ == "__main__":
    main()

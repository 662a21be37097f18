#!/usr/bin/env python
"""Kernel-variant sweep on one GPU (tuning aid, not the benchmark).

    python tools/tune.py --config 5 --variants "PARTS=1,PART_GROUP=2,PART_CSE=0;MODE=1"

Each variant is a set of PYRIT_B200_* knobs applied before the plan is compiled
(parts / part group / pair sharing / copy engine / tile) or the launch (mode).
Inputs are generated once on the device; every variant is timed with CUDA
events over --steps launches after --warmup launches and checked against the
first variant's output digest.  Prints one JSON line per variant.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--variants", required=True)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scale", type=int, default=1, help="divide the fragment size by this")
    ap.add_argument("--frag", type=int, default=0, help="fragment bytes (overrides the config's; > L2 working set)")
    ap.add_argument("--rounds", type=int, default=3, help="interleaved repeats per variant (median reported)")
    ap.add_argument("--no-graph", action="store_true", help="launch from Python instead of a captured CUDA graph")
    ap.add_argument("--code", default="", help="k,r,field[,transform]: an encode of this code instead of a config "
                    "(field gf16|gf64|gf256_r17|aop<w>; transform 0 embedding, 1 parity); needs --frag")
    a = ap.parse_args()

    import torch

    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200 import _lib as L
    from paper_1709_00178_b200.workloads import WORKLOADS

    lib = L.load()
    dev = torch.device("cuda", 0)
    transform = 0
    if a.code:
        from paper_1709_00178_b200.workloads import Workload
        parts = a.code.split(",")
        fn = parts[2]
        fld = P.FieldSpec.aop(int(fn[3:])) if fn.startswith("aop") else getattr(P.FieldSpec, fn + ("_aop" if fn == "gf16" else "_esp" if fn == "gf64" else ""))()
        transform = int(parts[3]) if len(parts) > 3 else 0
        wl = Workload(0, f"code-{a.code}", "encode", fld, int(parts[0]), int(parts[1]), a.frag, 7)
    else:
        wl = WORKLOADS[a.config]
    w = wl.fld.w
    S = (a.frag // w if a.frag else wl.strip // a.scale) // 16 * 16
    sym = w * S
    stream = torch.cuda.current_stream(dev).cuda_stream
    full = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, device=dev)
    for j in range(wl.k):
        for s in range(w):
            P.fill(full[j, s * S:(s + 1) * S], wl.seed, j, begin=s * wl.strip, valid=wl.valid)
    C = P.cauchy_parity_matrix(wl.code)
    enc = P.Plan.create(wl.fld, C)
    enc.apply([full[j].data_ptr() for j in range(wl.k)], [full[wl.k + i].data_ptr() for i in range(wl.m)], S,
              stream=stream)
    if wl.op == "encode":
        ins = [full[j].data_ptr() for j in range(wl.k)]
        out = torch.empty((wl.m, sym), dtype=torch.uint8, device=dev)
        outs = [out[i].data_ptr() for i in range(wl.m)]
        m = C
    else:
        surv, order, m = P.repair_matrix(wl.code, wl.erased)
        ins = [full[s].data_ptr() for s in surv]
        out = torch.empty((len(order), sym), dtype=torch.uint8, device=dev)
        outs = [out[i].data_ptr() for i in range(len(order))]
    moved = (len(ins) + len(outs)) * sym
    ref = None
    knobs = ("MODE", "COPY", "PARTS", "PART_GROUP", "PART_CSE", "PART_TEMPS", "THREADS", "LANES", "CSE_WINDOW", "WS")
    specs = a.variants.split(";")
    plans, graphs, times, clocks = {}, {}, {sp: [] for sp in specs}, {}
    for rnd in range(a.rounds):
        for spec in specs:
            env = dict(kv.split("=") for kv in spec.split(",") if kv)
            for k in knobs:
                os.environ.pop("PYRIT_B200_" + k, None)
            for k, v in env.items():
                os.environ["PYRIT_B200_" + k] = v
            L.check(lib.pyrit_set_kernel_mode(int(env.get("MODE", 0))))
            L.check(lib.pyrit_set_lanes(int(env.get("LANES", 1))))
            try:
                if spec not in plans:
                    plans[spec] = P.Plan.create(wl.fld, m, transform=transform)
                plan = plans[spec]
                for _ in range(a.warmup):
                    plan.apply(ins, outs, S, stream=stream)
                torch.cuda.synchronize()
                if not a.no_graph and spec not in graphs:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        cs = torch.cuda.current_stream().cuda_stream
                        for _ in range(a.steps):
                            plan.apply(ins, outs, S, stream=cs)
                    graphs[spec] = g
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                with ClockSampler(0) as clk:
                    e0.record()
                    if a.no_graph:
                        for _ in range(a.steps):
                            plan.apply(ins, outs, S, stream=stream)
                    else:
                        graphs[spec].replay()
                    e1.record()
                    torch.cuda.synchronize()
                clocks.setdefault(spec, []).append(clk.summary())
                times[spec].append(e0.elapsed_time(e1) / a.steps)
                if rnd == a.rounds - 1:
                    out.zero_()
                    plan.apply(ins, outs, S, stream=stream)
                    dg = int(P.digest(out).item())
                    if ref is None:
                        ref = dg
                    info = P.Plan.last_launch()
                    ts = sorted(times[spec])
                    ms = ts[len(ts) // 2]
                    print(json.dumps({"variant": spec, "key": plan.key(), "kernel": info["kernel"],
                                      "grid": [info["blocks"], info["threads"]], "ms": ms,
                                      "ms_all": [round(x, 5) for x in times[spec]],
                                      "moved_GBps": moved / ms / 1e6, "source_GBps": wl.k * sym / ms / 1e6,
                                      "frac_of_6452.8": moved / ms / 1e6 / 6452.8, "matches_first": dg == ref,
                                      "graph": not a.no_graph,
                                      "clocks": [(c["sm_mhz"], c["power_w_median"], c["reasons"]) for c in clocks[spec]]}), flush=True)
            except Exception as e:  # keep sweeping
                print(json.dumps({"variant": spec, "error": str(e)[:300]}), flush=True)
                times[spec] = times[spec] or [float("nan")]

if __name__ == "__main__":
    main()

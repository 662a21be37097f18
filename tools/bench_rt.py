#!/usr/bin/env python
"""Runtime-matrix ring kernel (ring_rt.cu) vs the generated specialised kernels.

    python tools/bench_rt.py [--configs 2,3,4,5] [--patterns N] [--reps R] [--out F.jsonl]

For each BASELINE config (full size, device resident, inputs > L2) time the
specialised kernel (kernel mode 0, prebuilt) and the runtime-matrix kernel
(kernel mode 4) with CUDA events on the launch stream, check the two outputs
are byte-identical, and print one JSON line per (config, kernel).  With
--patterns N, also time N random config-4 erasure patterns (data + parity) on
the runtime kernel on their FIRST launch (no compile), and the all-data worst
case {0,1,2,3}.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import sys

os.environ.setdefault("PYRIT_B200_TIERED", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200 import _lib as L  # noqa: E402
from paper_1709_00178_b200.workloads import WORKLOADS  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def setup(wl, dev):
    """(k+m) x frag buffer filled with the seeded generator; encode parity once."""
    buf = torch.empty((wl.k + wl.m, wl.frag), dtype=torch.uint8, device=dev)
    for j in range(wl.k):
        P.fill(buf[j], wl.seed, j, valid=wl.valid)
    buf[wl.k:] = 0
    return buf


def time_plan(plan, ins, outs, strip, reps, mode):
    lib = L.load()
    L.check(lib.pyrit_set_kernel_mode(mode))
    try:
        st = torch.cuda.current_stream().cuda_stream
        first0, first1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        first0.record()
        plan.apply(ins, outs, strip, stream=st)
        first1.record()
        torch.cuda.synchronize()
        kern = P.Plan.last_launch()["kernel"]
        for _ in range(2):
            plan.apply(ins, outs, strip, stream=st)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        for _ in range(reps):
            plan.apply(ins, outs, strip, stream=st)
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / reps, first0.elapsed_time(first1), kern
    finally:
        L.check(lib.pyrit_set_kernel_mode(0))


def run_config(cfg, dev, reps, out):
    wl = WORKLOADS[cfg]
    buf = setup(wl, dev)
    rows = [buf[j].data_ptr() for j in range(wl.k + wl.m)]
    if wl.op == "encode":
        plan = P.Plan.encode(wl.code)
        ins, outs = rows[: wl.k], rows[wl.k:]
        # encode once so decode-style checks have parity
    else:
        enc = P.Plan.encode(wl.code)
        enc.apply(rows[: wl.k], rows[wl.k:], wl.strip)
        plan = P.Plan.decode(wl.code, wl.erased)
        ins = [rows[s] for s in plan.survivors]
        outs = [rows[o] for o in plan.outputs]
    res = {}
    for name, mode in (("specialised", 0), ("ring_rt", 4)):
        out_rows = list(range(wl.k, wl.k + wl.m)) if wl.op == "encode" else list(plan.outputs)
        for o in out_rows:
            buf[o].zero_()
        ms, first_ms, kern = time_plan(plan, ins, outs, wl.strip, reps, mode)
        digest = [int(P.digest(buf[o]).item()) for o in out_rows]
        moved = wl.moved_bytes()
        gbs = moved / ms / 1e6
        line = {"cfg": cfg, "kernel": name, "name": kern, "ms": round(ms, 4), "first_ms": round(first_ms, 4),
                "moved_gbs": round(gbs, 1), "source_gbs": round(wl.source_bytes() / ms / 1e6, 1),
                "frac": round(gbs / peak(), 4), "digest": digest}
        res[name] = line
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")
    same = res["specialised"]["digest"] == res["ring_rt"]["digest"]
    print(json.dumps({"cfg": cfg, "outputs_identical": same}), flush=True)
    del buf
    torch.cuda.empty_cache()
    return same


def run_patterns(n, dev, reps, out, cfg=4):
    """Random erasure patterns of config 4 (or --pattern-config 5: the config-5 code) on the
    runtime kernel, first launch timed (never compiled)."""
    wl = WORKLOADS[cfg]
    buf = setup(wl, dev)
    rows = [buf[j].data_ptr() for j in range(wl.k + wl.m)]
    P.Plan.encode(wl.code).apply(rows[: wl.k], rows[wl.k:], wl.strip)
    ref = buf.clone()
    rng = random.Random(7)
    pats = [(0, 1, 2, 3), (1, 6, 9, 10)] + [tuple(sorted(rng.sample(range(wl.k + wl.m), 4))) for _ in range(n)]
    # one and two lost symbols (the common failures) and three
    pats += [(3,), (11,), (0, 7), (5, 12), (2, 4, 9)]
    jit0 = L.load().pyrit_jit_compiles()
    for er in pats:
        for o in er:
            buf[o].zero_()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        P.decode(buf, er, wl.code)  # policy default: ad-hoc pattern -> runtime kernel
        t1.record()
        torch.cuda.synchronize()
        first = t0.elapsed_time(t1)
        kern = P.Plan.last_launch()["kernel"]
        ok = bool(torch.equal(buf, ref))
        plan = P.Plan.decode(wl.code, er)
        ins = [rows[s] for s in plan.survivors]
        outs = [rows[o] for o in plan.outputs]
        ms, _, kern4 = time_plan(plan, ins, outs, wl.strip, reps, 4)
        moved = (wl.k + len(er)) * wl.frag
        line = {"pattern_cfg": cfg, "pattern": list(er), "first_call_ms": round(first, 4), "kernel_first": kern, "kernel_ms": round(ms, 4),
                "moved_gbs": round(moved / ms / 1e6, 1), "frac": round(moved / ms / 1e6 / peak(), 4),
                "repaired_ok": ok}
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")
        buf.copy_(ref)
    print(json.dumps({"patterns": len(pats), "nvrtc_compiles": L.load().pyrit_jit_compiles() - jit0}), flush=True)


def run_paper(dev, reps, out):
    """The paper's (60,40) GF(2^6)/R9 code (k=40, r=20; 4 MiB symbols): encode and a
    20-erasure decode on the specialised kernel vs the runtime-matrix kernel (one
    launch, three output groups)."""
    f = P.FieldSpec.gf64_esp()
    code = P.CodeSpec(40, 20, f, P.TransformKind.Embedding)
    strip = (4 << 20) // f.w // 16 * 16
    sym = f.w * strip
    buf = torch.empty((60, sym), dtype=torch.uint8, device=dev)
    for j in range(40):
        P.fill(buf[j], 7, j)
    rows = [buf[j].data_ptr() for j in range(60)]
    enc = P.Plan.encode(code)
    enc.apply(rows[:40], rows[40:], strip)
    torch.cuda.synchronize()
    ref = buf.clone()
    erased = tuple(range(20))
    dec = P.Plan.decode(code, erased)
    for label, plan, ins, outs, nmoved in (("encode", enc, rows[:40], rows[40:], 60),
                                           ("decode e=20", dec, [rows[s] for s in dec.survivors],
                                            [rows[o] for o in dec.outputs], 60)):
        res = {}
        # (a decode pattern never compiles in process: it runs the runtime kernel unless hot)
        kinds = (("specialised", 0), ("ring_rt", 4)) if label == "encode" else (("ring_rt", 4),)
        for name, mode in kinds:
            outs_idx = list(range(40, 60)) if label == "encode" else list(dec.outputs)
            for o in outs_idx:
                buf[o].zero_()
            ms, first_ms, kern = time_plan(plan, ins, outs, strip, reps, mode)
            ok = bool(torch.equal(buf, ref))
            gbs = nmoved * sym / ms / 1e6
            line = {"code": "(60,40) GF(2^6)", "op": label, "kernel": name, "name": kern, "ms": round(ms, 4),
                    "moved_gbs": round(gbs, 1), "source_gbs": round(40 * sym / ms / 1e6, 1),
                    "frac": round(gbs / peak(), 4), "exact": ok}
            res[name] = line
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")
    del buf
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--patterns", type=int, default=0)
    ap.add_argument("--pattern-config", type=int, default=4, choices=[4, 5],
                    help="the code whose erasure patterns --patterns draws (4: k10 m4 GF(2^8); 5: k16 m4 GF(2^12))")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--paper", action="store_true", help="also the paper's (60,40) GF(2^6) code")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = open(a.out, "a") if a.out else None
    ok = True
    for c in [int(x) for x in a.configs.split(",") if x]:
        ok &= run_config(c, dev, a.reps, out)
    if a.patterns:
        run_patterns(a.patterns, dev, a.reps, out, a.pattern_config)
    if a.paper:
        run_paper(dev, a.reps, out)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

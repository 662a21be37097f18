#!/usr/bin/env python
"""Host time per cached decode call on the GPU box.

    python tools/host_cost.py [--calls 2000]

Calls pyrit_cu_decode (device buffers, config-5 shape: k=16, m=4, GF(2^12),
4 erasures, 12 x 4 KiB strips so the GPU work is tiny and asynchronous) in a
loop and reports host microseconds per call, next to a no-op C-ABI call
(pyrit_kernel_launches) timed the same way to show the ctypes floor.  Also
times the first call of a new erasure pattern (repair matrix + light program).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    a = ap.parse_args()
    lib = L.load()
    code = P.CodeSpec(16, 4, P.FieldSpec.aop(12))
    ss = 12 * 4096
    dev = torch.device("cuda", 0)
    sym = torch.zeros((20, ss), dtype=torch.uint8, device=dev)
    rows = (C.c_void_p * 20)(*[sym[i].data_ptr() for i in range(20)])
    cc = code.c()
    stream = torch.cuda.current_stream().cuda_stream
    out = {}
    # first call of new patterns (host part: repair matrix, representatives, launch)
    firsts = []
    for er in [(0, 5, 16, 19), (1, 2, 3, 4), (3, 7, 11, 15), (0, 1, 18, 19)]:
        e = np.asarray(er, dtype=np.uint32)
        torch.cuda.synchronize()
        t = time.perf_counter()
        L.check(lib.pyrit_cu_decode(C.byref(cc), rows, e.ctypes.data, e.size, ss, stream))
        firsts.append((time.perf_counter() - t) * 1e6)
    out["first_call_us"] = [round(x, 1) for x in firsts]
    e = np.asarray((0, 5, 16, 19), dtype=np.uint32)
    ep = e.ctypes.data
    for _ in range(50):
        lib.pyrit_cu_decode(C.byref(cc), rows, ep, 4, ss, stream)
    torch.cuda.synchronize()
    n = a.calls

    def host_us(fn):
        """median host time per call over batches of 64 enqueues (a sync before each
        batch, none inside: the launch queue never fills, so this is host work only)"""
        per = []
        for _ in range(max(1, n // 64)):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(64):
                fn()
            per.append((time.perf_counter() - t) / 64 * 1e6)
        per.sort()
        return per[len(per) // 2]

    ccr = C.byref(cc)
    host = host_us(lambda: lib.pyrit_cu_decode(ccr, rows, ep, 4, ss, stream))
    floor = host_us(lambda: lib.pyrit_kernel_launches())
    # the same launch through a decode plan (no decode_program lookup) and the
    # specialised encode kernel (small parameter block) for comparison
    plan = P.Plan.decode(code, (0, 5, 16, 19))
    ins = (C.c_void_p * 16)(*[sym[s].data_ptr() for s in plan.survivors])
    outs = (C.c_void_p * 4)(*[sym[o].data_ptr() for o in plan.outputs])
    for _ in range(50):
        lib.pyrit_cu_apply(plan._h, ins, outs, 4096, 0, 4096, stream)
    apply_us = host_us(lambda: lib.pyrit_cu_apply(plan._h, ins, outs, 4096, 0, 4096, stream))
    torch.cuda.synchronize()
    enc = P.Plan.encode(code)
    ein = (C.c_void_p * 16)(*[sym[j].data_ptr() for j in range(16)])
    eout = (C.c_void_p * 4)(*[sym[16 + i].data_ptr() for i in range(4)])
    for _ in range(50):
        lib.pyrit_cu_apply(enc._h, ein, eout, 4096, 0, 4096, stream)
    enc_us = host_us(lambda: lib.pyrit_cu_apply(enc._h, ein, eout, 4096, 0, 4096, stream))
    enc_kernel = P.Plan.last_launch()["kernel"]
    torch.cuda.synchronize()
    out.update({"cached_decode_host_us": round(host, 2), "ctypes_noop_us": round(floor, 2),
                "apply_decode_plan_us": round(apply_us, 2), "apply_encode_plan_us": round(enc_us, 2),
                "encode_kernel": enc_kernel,
                "cached_decode_minus_ctypes_us": round(host - floor, 2),
                "kernel": P.Plan.last_launch()["kernel"], "shape": "k16 m4 GF(2^12) R13, 4 erased, 12 x 4 KiB strips"})
    print(json.dumps(out))


if __name__ == "__main__":
    main()

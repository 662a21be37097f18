#!/usr/bin/env python
"""Compile latency of the specialised kernels ("NVRTC compile latency per plan is reported").

    python tools/jit_latency.py [--tiered] [--out F.jsonl]

With no prebuilt kernels (an empty PYRIT_B200_KERNEL_DIR) and no disk cache
(PYRIT_B200_JIT_CACHE=0), each program's first launch compiles its kernel:
  * default: in process (PYRIT_B200_TIERED=0), so the launch waits for NVRTC;
  * --tiered: the first launch runs the runtime-matrix kernel while the helper
    process compiles; pyrit_jit_wait() then waits for the helper.
pyrit_jit_time() reports the wall time of each compile.  Programs: the five
BASELINE encodes at their kernel shapes (4 MiB strips: the staged kernels), the
config-4 decode patterns, a config-5 decode pattern, and the paper's (60,40)
GF(2^6) code.  One JSON line per program.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import tempfile
import time

ap = argparse.ArgumentParser()
ap.add_argument("--tiered", action="store_true")
ap.add_argument("--out", default="")
a = ap.parse_args()
os.environ["PYRIT_B200_KERNEL_DIR"] = tempfile.mkdtemp(prefix="pyrit_nokernels_")
os.environ["PYRIT_B200_JIT_CACHE"] = "0"
os.environ["PYRIT_B200_TIERED"] = "1" if a.tiered else "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200 import _lib as L  # noqa: E402
from paper_1709_00178_b200.workloads import WORKLOADS  # noqa: E402


def jit_ms():
    last, total = C.c_double(), C.c_double()
    L.check(L.load().pyrit_jit_time(C.byref(last), C.byref(total)))
    return last.value, total.value


def main():
    lib = L.load()
    L.check(lib.pyrit_set_kernel_dir(os.environ["PYRIT_B200_KERNEL_DIR"].encode()))
    dev = torch.device("cuda", 0)
    progs = []
    for c in (1, 2, 3, 5):
        progs.append((f"cfg{c} encode", WORKLOADS[c].code, None))
    progs.append(("cfg4 decode {1,6,9,10}", WORKLOADS[4].code, (1, 6, 9, 10)))
    progs.append(("cfg4 decode {0,1,2,3}", WORKLOADS[4].code, (0, 1, 2, 3)))
    progs.append(("cfg5 decode {2,7,11,17}", WORKLOADS[5].code, (2, 7, 11, 17)))
    progs.append(("(60,40) GF(2^6) encode", P.CodeSpec(40, 20, P.FieldSpec.gf64_esp(), P.TransformKind.Embedding), None))
    # warm-up: the first compile of a process on a fresh box also pages in NVRTC and
    # its builtins (100-400 ms extra); compile one small unrelated program first so the
    # lines below are steady-state, and report that first compile separately
    if True:
        wcode = P.CodeSpec(3, 2, P.FieldSpec.gf16_aop(), P.TransformKind.Embedding)
        wplan = P.Plan.encode(wcode)
        wbuf = torch.zeros((5, 4 * (1 << 20)), dtype=torch.uint8, device=dev)
        h0 = time.perf_counter()
        wplan.apply([wbuf[j].data_ptr() for j in range(3)], [wbuf[3 + i].data_ptr() for i in range(2)], 1 << 20)
        L.check(lib.pyrit_jit_wait())
        torch.cuda.synchronize()
        warm = {"program": "warm-up (3,2) GF(2^4) encode, first compile of the process", "tiered": a.tiered,
                "compile_ms": round(jit_ms()[0], 1), "wall_ms": round((time.perf_counter() - h0) * 1e3, 1)}
        print(json.dumps(warm), flush=True)
        del wbuf
    out = open(a.out, "a") if a.out else None
    for name, code, erased in progs:
        w = code.field.w
        strip = 4 << 20
        plan = P.Plan.encode(code) if erased is None else P.Plan.decode(code, erased)
        nin = code.k
        nout = code.r if erased is None else len(erased)
        buf = torch.zeros((nin + nout, w * strip), dtype=torch.uint8, device=dev)
        ins = [buf[j].data_ptr() for j in range(nin)]
        outs = [buf[nin + i].data_ptr() for i in range(nout)]
        n0 = lib.pyrit_jit_compiles()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # decode patterns run on the runtime-matrix kernel until one is hot: force
        # the specialised kernel (kernel mode 2) in process, or make it hot (8
        # launches, PYRIT_B200_HOT_PATTERN) with tiered compilation
        if erased is not None and not a.tiered:
            L.check(lib.pyrit_set_kernel_mode(2))
        h0 = time.perf_counter()
        plan.apply(ins, outs, strip)
        first_kernel = P.Plan.last_launch()["kernel"]
        h1 = time.perf_counter()
        if erased is not None and a.tiered:
            for _ in range(7):
                plan.apply(ins, outs, strip)
        L.check(lib.pyrit_jit_wait())
        h2 = time.perf_counter()
        torch.cuda.synchronize()
        plan.apply(ins, outs, strip)
        torch.cuda.synchronize()
        L.check(lib.pyrit_set_kernel_mode(0))
        last, _ = jit_ms()
        line = {"program": name, "tiered": a.tiered, "compiles": lib.pyrit_jit_compiles() - n0,
                "compile_ms": round(last, 1), "first_call_host_ms": round((h1 - h0) * 1e3, 2),
                "wait_ms": round((h2 - h1) * 1e3, 1), "first_kernel": first_kernel,
                "kernel": P.Plan.last_launch()["kernel"]}
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")
        del buf
        plan.close()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

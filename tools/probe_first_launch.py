#!/usr/bin/env python
"""First-launch cost of the runtime-matrix kernel in a fresh process: wall time of the first
decode of new erasure patterns (one lost symbol, then two, then four) on config-4 shaped
symbols, each a kernel instance not yet used in this process, and of a second pattern of each
size (instance already loaded)."""
import json
import os
import sys
import time

os.environ.setdefault("PYRIT_B200_TIERED", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1709_00178_b200 as P  # noqa: E402
from paper_1709_00178_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[4]
dev = torch.device("cuda", 0)
t_start = time.perf_counter()
full = torch.zeros((wl.k + wl.m, wl.fld.w * 4096), dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
res = {"module_loading": os.environ.get("CUDA_MODULE_LOADING", "default(lazy)"),
       "torch_setup_ms": round((time.perf_counter() - t_start) * 1e3, 1)}
t0 = time.perf_counter()
P.gf_mul(3, 5, wl.fld)  # loads the library (host only)
res["load_library_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
t0 = time.perf_counter()
P.encode(full[: wl.k], wl.code)  # the library's first device work (its CUDA runtime, a prebuilt kernel)
torch.cuda.synchronize()
res["first_encode_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
if os.environ.get("PROBE_WARMUP") == "1":
    from paper_1709_00178_b200 import _lib as L
    t0 = time.perf_counter()
    L.check(L.load().pyrit_warmup(0))
    res["warmup_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
for name, pats in (("one", [(3,), (7,)]), ("two", [(0, 7), (5, 12)]), ("four", [(2, 5, 6, 10), (0, 1, 8, 12)])):
    for q, er in enumerate(pats):
        t0 = time.perf_counter()
        P.decode(full, er, wl.code)
        torch.cuda.synchronize()
        res[f"{name}_{'first' if q == 0 else 'second'}_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
        res[f"{name}_kernel"] = P.Plan.last_launch()["kernel"]
print(json.dumps(res))

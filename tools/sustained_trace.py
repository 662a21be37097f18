#!/usr/bin/env python
"""Launch-by-launch trace of a BASELINE config's kernel (sustained behaviour).

    CFG=5 N=300 python tools/sustained_trace.py

Launches the encode program N times back to back from Python, records a CUDA event
after every launch, and prints one JSON line. The line has the mean launch time over
launches 0-19, 20-99 and 100-end, and every 10th launch time. These traces are the
sustained_trace_* files under profiles/r01_s2: they compare the TMA and cp.async
producers, and the torch copy probes.
"""
import os, sys, json, time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in
sys.path.insert(0, os.getcwd())
import torch
import paper_1709_00178_b200 as P
from paper_1709_00178_b200.workloads import WORKLOADS
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
wl = WORKLOADS[int(os.environ.get("CFG", "5"))]; w = wl.fld.w; Ls = wl.strip; sym = w * Ls
data = torch.empty((wl.k, sym), dtype=torch.uint8, device=dev)
for j in range(wl.k):
    for s in range(w):
        P.fill(data[j][s*Ls:(s+1)*Ls], wl.seed, j, begin=s*wl.strip, valid=wl.valid)
par = torch.empty((wl.m, sym), dtype=torch.uint8, device=dev)
ins = [data[j].data_ptr() for j in range(wl.k)]; outs = [par[i].data_ptr() for i in range(wl.m)]
stream = torch.cuda.current_stream(dev).cuda_stream
plan = P.Plan.create(wl.fld, P.cauchy_parity_matrix(wl.code))
for _ in range(3): plan.apply(ins, outs, Ls, stream=stream)
torch.cuda.synchronize()
n = int(os.environ.get("N", "300"))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
ev[0].record()
for i in range(n):
    plan.apply(ins, outs, Ls, stream=stream); ev[i + 1].record()
torch.cuda.synchronize()
t = [round(ev[i].elapsed_time(ev[i + 1]), 4) for i in range(n)]
dg = int(P.digest(par).item())
print(json.dumps({"copy": os.environ.get("PYRIT_B200_COPY", "1"), "cfg": wl.cfg, "kernel": P.Plan.last_launch()["kernel"], "digest": dg, "first20": sum(t[:20]) / 20, "20-100": sum(t[20:100]) / 80, "100-end": sum(t[100:]) / max(1, n - 100), "trace": t[::10]}))

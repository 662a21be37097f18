#!/usr/bin/env python
"""PYRIT ring-codec benchmark on B200 (see DESIGN.md section "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl b200|reference]

One step = one pass of the fused encode (or decode) kernel over this rank's
byte-offset shard of every strip of the workload (BASELINE.json config 5 by
default: GF(2^12) in R_{2,13}, k=16, m=4, 512 MiB fragments, 8 GiB of source
sharded across the N GPUs -- total work fixed, so scaling is "strong").
`value` = source bytes of the whole job / max-over-ranks device time (inputs
resident in HBM, larger than L2; smaller workloads rotate buffer sets so the
working set exceeds L2).  `e2e` = the same metric through the public
host-buffer C ABI (pyrit_encode_host / pyrit_decode_host) with pinned host
buffers, H2D and D2H inside the timed region.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PYRIT encode/decode GB/s (source bytes) at 1/2/4/8 B200; % of HBM roofline"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device: int, interval_ms: int = 100):
        self.device = device
        self.interval_ms = interval_ms
        self.rows = []
        self.proc = None
        self.thread = None
        self.first = threading.Event()

    def __enter__(self):
        # nvidia-smi's start-up (NVML initialisation) perturbs the GPU for a
        # few hundred ms -- measured: +10% on a 35 ms timed region -- so the
        # sampler is started first and the caller's timed region begins only
        # once the first sample has arrived (the recipe's "start before")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            self.first.wait(timeout=5.0)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)
                self.first.set()

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0, "power_w_median": None}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        pw = [float(r[7]) for r in self.rows if r[7].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_median": statistics.median(pw) if pw else None}


def cpu_baseline(wl, steps=None, warmup=1, budget_s=12.0, sample_frag=None):
    """Reference CPU path (oracle/_ref, the unmodified reference headers) on a bounded sample."""
    import numpy as np

    import oracle as O

    threads = os.cpu_count() or 1
    f = O.Field(wl.fld.w, wl.fld.n, wl.fld.kind, wl.fld.s, wl.fld.r_esp or wl.fld.w, wl.fld.modulus)
    q = 16 * wl.fld.w
    frag = sample_frag or min(wl.frag, max(q, (16 << 20) // q * q))
    # ring schedule where the reference's ring path is valid (AOP/ESP moduli);
    # CRS bitmatrix schedule for R_{2,17} (the reference's ring path truncates
    # 17-bit ring elements); decode = decode_matrix + CRS passes
    aop_esp = wl.fld.n <= 16
    mode = (0 if aop_esp else 1) if wl.op == "encode" else (3 if aop_esp else 2)
    kind = "reference"
    try:
        plan = O.RefPlan(f, wl.k, wl.m, mode, frag, wl.erased)
    except Exception:
        plan = None
    if plan is None:
        return None
    # seeded bytes: a 16 MiB block of uniform bytes tiled over every symbol (the
    # CPU kernel's speed does not depend on the values; filling 10 GiB of full
    # config-5 buffers byte by byte from the generator would dominate the run)
    blk = np.frombuffer(np.random.default_rng(wl.seed).bytes(min(frag, 16 << 20)), dtype=np.uint8)
    for s in range(wl.k + wl.m):
        v = plan.symbol(s)
        for o in range(0, frag, blk.size):
            v[o:o + blk.size] = blk[: min(blk.size, frag - o)]
    for _ in range(warmup):
        plan.run(threads)
    times = []
    t_start = time.perf_counter()
    n = 0
    while True:
        t0 = time.perf_counter()
        plan.run(threads)
        times.append(time.perf_counter() - t0)
        n += 1
        if steps is not None and n >= steps:
            break
        if steps is None and (time.perf_counter() - t_start > budget_s or n >= 50):
            break
    # one thread as well (T = hardware threads and T = 1), a few runs
    t1 = []
    if steps is None:
        for _ in range(3):
            t0 = time.perf_counter()
            plan.run(1)
            t1.append(time.perf_counter() - t0)
    plan.close()
    src = wl.k * frag
    t = statistics.median(times)
    names = {0: "ring schedule (compile_schedule + parallel_replay)",
             1: "CRS bitmatrix schedule (compile_crs_schedule + parallel_replay)",
             2: "decode_matrix + CRS parallel_replay, then CRS parity rows (decode() restated)",
             3: "decode_matrix + ring parallel_replay, then ring parity rows (decode())"}
    extra = {"value_1_thread": src / min(t1) / 1e9} if t1 else {}
    # the reference bench's own convention counts (k + r) * F bytes (bench.hpp:205-207)
    extra["value_kr_convention"] = (wl.k + wl.m) * frag / t / 1e9
    return {"value": src / t / 1e9, "unit": "GB/s", "cores": threads, "kind": kind, **extra, "fragment_bytes": frag,
            "sample": f"{wl.k}x{frag}-byte fragments ({src / 2**20:.0f} MiB source) of the {wl.name} shape, "
                      f"{names[mode]}, {threads} threads, median of {len(times)} runs",
            "times_s": [round(x, 5) for x in times]}


def run_reference(args, rank, world):
    from paper_1709_00178_b200.workloads import WORKLOADS
    if rank != 0:
        return 0
    wl = WORKLOADS[args.config]
    # the full BASELINE workload every step (same_config): config 5 is 8 GiB of
    # source per parallel_replay pass, ~2 s on the box's 16 host threads
    res = cpu_baseline(wl, steps=args.steps, warmup=min(args.warmup, 1), sample_frag=wl.frag)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpyrit_ref.so not built"}))
        return 0
    times = res.pop("times_s")
    ms = statistics.mean(times) * 1e3
    line = {"metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": world, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded uniform bytes)",
            "config": {"workload": wl.name, "fragment_bytes": res.get("fragment_bytes"),
                       "same_config": res.get("fragment_bytes") == wl.frag}, "impl": "reference",
            "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def dry_run(args, rank, world) -> int:
    """PYRIT_B200_BENCH_DRYRUN=1: the rank plumbing only (no GPU work), on gloo --
    what tests/test_bench_cli.py checks on CPU: every rank joins one group."""
    import torch
    import torch.distributed as dist
    n = 1
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dryrun": True, "world_size": world, "comm_nranks": n, "requested_gpus": args.gpus,
                          "spawned_by_bench": os.environ.get("PYRIT_B200_SPAWNED") == "1"}), flush=True)
    return 0


def spawn_ranks(n: int, argv) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks of this script with
    torch.distributed.run on 127.0.0.1 (one process per GPU, NCCL); rank 0's
    JSON line is this process's output.  NCCL's init log goes to stderr."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if env.get("PYRIT_B200_DIST_BACKEND", "nccl") == "nccl" and env.get("PYRIT_B200_BENCH_DRYRUN") != "1":
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env["PYRIT_B200_SPAWNED"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    print("bench.py: spawning", n, "ranks:", " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps from Python")
    ap.add_argument("--erased", default="", help="decode configs: erased symbols, e.g. 0,1,2,3 (config 4's "
                                                 "all-data worst case; default: the BASELINE pattern)")
    args = ap.parse_args(argv)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "b200":
        # one process per GPU: re-run this command under torchrun (the driver may
        # launch `bench.py --gpus N` directly or under torchrun itself)
        return spawn_ranks(args.gpus, sys.argv[1:] if argv is None else list(argv))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, max(world, args.gpus))
    if os.environ.get("PYRIT_B200_BENCH_DRYRUN") == "1":
        return dry_run(args, rank, world)
    if args.warmup < 3:
        args.warmup = 3  # contract: at least 3 warm-up steps

    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200 import _lib as L
    from paper_1709_00178_b200.workloads import WORKLOADS, shard

    # PYRIT_B200_DIST_BACKEND=gloo: harness check of the N-rank path on a box with
    # fewer GPUs (ranks share devices round-robin; shards are independent, only
    # the scalar timing reduction and the digest gather cross ranks, over gloo)
    backend = os.environ.get("PYRIT_B200_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # where collective tensors live
    ranks = {"world_size": world, "requested_gpus": args.gpus, "backend": backend if world > 1 else None,
             "spawned_by_bench": os.environ.get("PYRIT_B200_SPAWNED") == "1"}
    if world > 1:
        one = torch.ones(1, dtype=torch.float64, device=cdev)
        dist.all_reduce(one)  # every rank joined the communicator
        ranks["comm_nranks"] = int(one.item())
        dl = [None] * world
        dist.all_gather_object(dl, {"rank": rank, "device": torch.cuda.current_device(),
                                    "name": torch.cuda.get_device_name(dev)})
        ranks["devices"] = dl
    ranks["ok"] = world == args.gpus and ranks.get("comm_nranks", 1) == world
    lib = L.load()
    if args.lanes:
        L.check(lib.pyrit_set_lanes(args.lanes))
    wl = WORKLOADS[args.config]
    if args.erased and wl.op == "decode":
        import dataclasses
        er = tuple(int(x) for x in args.erased.split(","))
        wl = dataclasses.replace(wl, erased=er, name=wl.name.rsplit("-e", 1)[0] + "-e" + ",".join(map(str, er)))
    w = wl.fld.w
    lo, hi = shard(wl.strip, rank, world)
    Ls = hi - lo
    n_in, n_out = wl.k, wl.n_out
    sym = w * Ls  # the shard of every fragment is itself a SymbolBuffer of w strips of Ls bytes
    stream = torch.cuda.current_stream(dev)

    def fill_symbol(t, frag):
        for s in range(w):
            P.fill(t[s * Ls:(s + 1) * Ls], wl.seed, frag, begin=s * wl.strip + lo, valid=wl.valid)

    # ---- device-resident inputs (rotating sets when one set fits in L2)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    moved_rank = (n_in + n_out) * sym
    nsets = 1 if moved_rank >= 4 * l2 else -(-4 * l2 // moved_rank)
    code = wl.code
    if wl.op == "encode":
        plan = P.Plan.encode(code)
        sets = []
        for _ in range(nsets):
            data = torch.empty((wl.k, sym), dtype=torch.uint8, device=dev)
            for j in range(wl.k):
                fill_symbol(data[j], j)
            par = torch.empty((wl.m, sym), dtype=torch.uint8, device=dev)
            sets.append(([data[j].data_ptr() for j in range(wl.k)], [par[i].data_ptr() for i in range(wl.m)],
                         data, par))
    else:
        enc = P.Plan.encode(code)
        plan = P.Plan.decode(code, wl.erased)
        sets = []
        for _ in range(nsets):
            full = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, device=dev)
            for j in range(wl.k):
                fill_symbol(full[j], j)
            enc.apply([full[j].data_ptr() for j in range(wl.k)],
                      [full[wl.k + i].data_ptr() for i in range(wl.m)], Ls, stream=stream.cuda_stream)
            sets.append(([full[s].data_ptr() for s in plan.survivors], [full[o].data_ptr() for o in plan.outputs],
                         full, None))
    torch.cuda.synchronize(dev)

    def step(i):
        ins, outs = sets[i % nsets][0], sets[i % nsets][1]
        plan.apply(ins, outs, Ls, 0, Ls, stream=stream.cuda_stream)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    # the K timed steps are captured once into a CUDA graph (one kernel node per
    # step) so that small configurations are not bound by Python launch overhead
    graph = None
    launches0 = lib.pyrit_kernel_launches()
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            cs = torch.cuda.current_stream().cuda_stream
            for i in range(args.steps):
                ins, outs = sets[i % nsets][0], sets[i % nsets][1]
                plan.apply(ins, outs, Ls, 0, Ls, stream=cs)
        torch.cuda.synchronize(dev)
        graph.replay()  # untimed replay (graph upload)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(i)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    launches = args.steps if graph is not None else lib.pyrit_kernel_launches() - launches0
    launch = P.Plan.last_launch()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = wl.source_bytes() / (ms_max * 1e-3) / 1e9

    # ---- self-check outside the timed region: erase 4 data symbols (or, for
    # decode, compare against the pre-erasure symbols) and repair on the GPU;
    # digests of repaired vs original bytes must match on every rank (K3 digests
    # gathered over NCCL -- the only collective, verification only).
    verified = verify(P, wl, plan, sets[0], sym, Ls, dev, stream, world)
    refcheck = verify_reference(wl, plan, sets[0], sym, Ls, dev, world)

    # ---- end to end through the public host-buffer API
    e2e = None
    e2e_dev = None
    if not args.no_e2e:
        e2e = run_e2e(P, wl, sets[0], sym, Ls, dev, world, args.e2e_steps or min(args.steps, 10))
        if world > 1:
            e2e_dev = run_e2e_devices(P, wl, world, rank, args.e2e_steps or min(args.steps, 10))

    peak, peak_src = measured_peaks()
    rt_probe = runtime_matrix_probe(P, L, wl, sets[0], sym, Ls, dev, stream, peak) if rank == 0 else None
    alg_bytes = (n_in + n_out) * sym
    achieved = alg_bytes / (ms * 1e-3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)
        if cpu:
            cpu.pop("times_s", None)
    st = plan.stats()
    if rank == 0:
        # ncu DRAM bytes of THIS kernel at this shard size (profiles/traffic.json is keyed by
        # kernel name; a kernel the table has not seen reports null, never a stale number)
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                ent = json.load(f).get("kernels", {}).get(f"{launch['kernel']}|{Ls}")
            traffic = ent["traffic_bytes"] if ent else None
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded uniform bytes, counter-based mix64)",
            "config": {"workload": wl.name, "op": wl.op, "k": wl.k, "m": wl.m, "w": w, "n": wl.fld.n,
                       "p": hex(wl.fld.modulus), "fragment_bytes": wl.frag, "strip_bytes": wl.strip,
                       "shard_strip_bytes": Ls, "erased": list(wl.erased), "parallelism": f"byte-offset shards x{world}",
                       "l2": "inputs larger than L2" if nsets == 1 else f"{nsets} rotating buffer sets > L2",
                       "launch": "CUDA graph of the K steps" if graph is not None else "per-step launches",
                       "kernel": launch["kernel"], "grid": [launch["blocks"], launch["threads"]],
                       "xors_per_column_word": st["part_xors"] if ("_cpa" in launch["kernel"] or "_tm" in
                                                                   launch["kernel"]) else st["xors"],
                       "reference_region_ops": st["ref_region_ops"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg_bytes, "launch_ms": ms,
                         "frac_of_8TBps_nominal": achieved / 8000.0},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": int(launches),
            "verified": bool(refcheck["identical"]) if refcheck.get("identical") is not None else verified,
            "verification": {"reference": refcheck, "repair_round_trip": verified},
            "ranks": ranks,
        }
        if e2e_dev is not None:
            line["e2e_devices"] = e2e_dev
        if rt_probe is not None:
            line["runtime_matrix"] = rt_probe
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def runtime_matrix_probe(P, L, wl, s0, sym, Ls, dev, stream, peak):
    """Outside the timed region: a decode of an erasure pattern this process has never seen
    (no prebuilt or compiled kernel) on rank 0's shard -- what a new failure costs: it runs on
    the runtime-matrix ring kernel (csrc/ring_rt.cu, the matrix in kernel parameters) with no
    compile.  First launch (plan + launch) and the mean of 5 more, CUDA events on the stream;
    the repaired symbols must equal the originals."""
    import torch
    try:
        lib = L.load()
        full = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, device=dev)
        if wl.op == "encode":
            full[: wl.k].copy_(s0[2])
            full[wl.k:].copy_(s0[3])
            erased = list(range(wl.k - min(wl.m, 4), wl.k))  # the last data symbols
        else:
            full.copy_(s0[2])
            erased = [2, 5, 6, wl.k]  # not the benchmarked pattern
        ref = [P.digest(full[e]) for e in erased]
        plan = P.Plan.decode(wl.code, erased)
        ins = [full[x].data_ptr() for x in plan.survivors]
        outs = [full[o].data_ptr() for o in plan.outputs]
        jit0 = lib.pyrit_jit_compiles()
        full[erased] = 0xA5
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        h0 = time.perf_counter()
        plan.apply(ins, outs, Ls, stream=stream.cuda_stream)
        host_ms = (time.perf_counter() - h0) * 1e3
        ev[1].record(stream)
        kern = P.Plan.last_launch()["kernel"]
        ev[2].record(stream)
        for _ in range(5):
            plan.apply(ins, outs, Ls, stream=stream.cuda_stream)
        ev[3].record(stream)
        torch.cuda.synchronize(dev)
        exact = all(int(P.digest(full[e]).item()) == int(r.item()) for e, r in zip(erased, ref))
        ms = ev[2].elapsed_time(ev[3]) / 5
        moved = (wl.k + len(erased)) * sym
        res = {"pattern": erased, "kernel": kern, "first_launch_ms": round(ev[0].elapsed_time(ev[1]), 4),
               "first_call_host_ms": round(host_ms, 3),
               "ms": round(ms, 4), "source_GBps": round(wl.k * sym / ms / 1e6, 1),
               "frac": round(moved / ms / 1e6 / peak, 4), "exact": exact,
               "nvrtc_compiles": int(lib.pyrit_jit_compiles() - jit0)}
        del full
        torch.cuda.empty_cache()
        return res
    except Exception as e:  # a probe, never the bench's failure
        return {"error": str(e)[:200]}


def verify(P, wl, plan, s0, sym, Ls, dev, stream, world):
    import torch
    import torch.distributed as dist
    ok = True
    if wl.op == "encode":
        full = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, device=dev)
        full[: wl.k].copy_(s0[2])
        full[wl.k:].copy_(s0[3])
        erase = list(range(min(wl.m, wl.k)))
        ref = [P.digest(full[e]) for e in erase]
        dplan = P.Plan.decode(wl.code, erase)
        full[erase] = 0xA5
        dplan.apply([full[s].data_ptr() for s in dplan.survivors], [full[o].data_ptr() for o in dplan.outputs],
                    Ls, stream=stream.cuda_stream)
        got = [P.digest(full[e]) for e in erase]
    else:
        full = s0[2]
        ref = [P.digest(full[o]) for o in plan.outputs]  # repaired in the timed loop
        saved = full[plan.outputs].clone()
        full[plan.outputs] = 0x5A
        plan.apply([full[s].data_ptr() for s in plan.survivors], [full[o].data_ptr() for o in plan.outputs], Ls,
                   stream=stream.cuda_stream)
        got = [P.digest(full[o]) for o in plan.outputs]
        ok = bool(torch.equal(saved, full[plan.outputs]))
    dg = torch.cat([torch.cat(ref), torch.cat(got)])
    if world > 1:
        if os.environ.get("PYRIT_B200_DIST_BACKEND", "nccl") != "nccl":
            dg = dg.cpu()
        allg = [torch.empty_like(dg) for _ in range(world)]
        dist.all_gather(allg, dg)
        dg = torch.stack(allg)
    dg = dg.view(-1, 2, len(ref))
    return bool(ok and torch.equal(dg[:, 0], dg[:, 1]))


def verify_reference(wl, plan, s0, sym, Ls, dev, world):
    """Every output byte of this rank's shard against the reference's own CPU
    output on the same input bytes: oracle/_ref (the unmodified reference
    headers), parallel_replay of the reference's schedule over all host threads
    -- the ring schedule for AOP fields, the CRS schedule for R_{2,17} where the
    reference's ring path is wrong; for decode, decode() restated
    over the survivors the GPU decoded from.  Outside the timed region."""
    import numpy as np
    import torch
    try:
        import oracle as O
        f = O.Field(wl.fld.w, wl.fld.n, wl.fld.kind, wl.fld.s, wl.fld.r_esp or wl.fld.w, wl.fld.modulus)
        aop_esp = wl.fld.n <= 16
        mode = (0 if aop_esp else 1) if wl.op == "encode" else (3 if aop_esp else 2)
        ref = O.RefPlan(f, wl.k, wl.m, mode, sym, wl.erased)
    except Exception as e:  # no reference build on this box
        return {"identical": None, "why": f"reference unavailable: {e}"}
    t0 = time.perf_counter()
    try:
        full = s0[2]
        if wl.op == "encode":
            for j in range(wl.k):
                torch.from_numpy(ref.symbol(j)).copy_(full[j])
            outs = list(range(wl.k, wl.k + wl.m))
            gpu = {wl.k + i: s0[3][i] for i in range(wl.m)}
        else:
            # the GPU repaired full[outputs] in place from full[survivors]
            for s in plan.survivors:
                torch.from_numpy(ref.symbol(s)).copy_(full[s])
            outs = list(plan.outputs)
            gpu = {o: full[o] for o in outs}
        torch.cuda.synchronize(dev)
        ref.run(os.cpu_count() or 1)
        same = True
        host = torch.empty(sym, dtype=torch.uint8, pin_memory=True)
        for o in outs:
            host.copy_(gpu[o])
            same &= bool(np.array_equal(host.numpy(), ref.symbol(o)))
        return {"identical": same, "bytes_compared": len(outs) * sym,
                "reference": ("ring schedule" if mode in (0, 3) else "CRS schedule") + " parallel_replay"
                             + (" + decode()" if wl.op == "decode" else ""),
                "threads": os.cpu_count(), "seconds": round(time.perf_counter() - t0, 2),
                "scope": f"rank shard: {len(outs)} outputs x {sym} bytes"}
    finally:
        ref.close()


def run_e2e_devices(P, wl, world, rank, steps):
    """The library's own multi-device path: rank 0 calls pyrit_encode_host_devices /
    pyrit_decode_host_devices over devices 0..N-1 on the WHOLE workload (byte-offset
    shards, one host thread + staging ring per device) while the other ranks wait."""
    import numpy as np
    import torch
    import torch.distributed as dist
    res = None
    if rank == 0:
        try:
            sym = wl.frag
            devs = [i % torch.cuda.device_count() for i in range(world)]  # gloo harness: ranks share GPUs
            blk = np.frombuffer(np.random.default_rng(wl.seed).bytes(16 << 20), dtype=np.uint8)
            if wl.op == "encode":
                host_in = torch.empty((wl.k, sym), dtype=torch.uint8, pin_memory=True)
                host_out = torch.empty((wl.m, sym), dtype=torch.uint8, pin_memory=True)
                a_in, a_out = host_in.numpy(), host_out.numpy()
                flat = a_in.reshape(-1)
                for o in range(0, flat.size, blk.size):
                    flat[o:o + blk.size] = blk[: min(blk.size, flat.size - o)]

                def call():
                    P.encode_host(a_in, wl.code, parity=a_out, devices=devs)
                h2d, d2h = wl.k * sym, wl.m * sym
            else:
                host = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, pin_memory=True)
                a = host.numpy()
                flat = a.reshape(-1)
                for o in range(0, flat.size, blk.size):
                    flat[o:o + blk.size] = blk[: min(blk.size, flat.size - o)]

                def call():
                    P.decode_host(a, wl.erased, wl.code, devices=devs)
                h2d, d2h = wl.k * sym, len(wl.erased) * sym
            call()
            times = []
            for _ in range(max(2, steps // 2)):
                t0 = time.perf_counter()
                call()
                times.append(time.perf_counter() - t0)
            t = statistics.median(times)
            res = {"value": wl.source_bytes() / t / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": t * 1e3, "steps": len(times),
                   "api": ("pyrit_encode_host_devices" if wl.op == "encode" else "pyrit_decode_host_devices")
                          + f" over devices {devs} from rank 0 (one process)",
                   "data": "16 MiB seeded block tiled (pinned host buffers)"}
            del flat
        except Exception as e:
            res = {"error": str(e)[:300]}
    dist.barrier()
    return res


def run_e2e(P, wl, s0, sym, Ls, dev, world, steps):
    import torch
    import torch.distributed as dist
    from paper_1709_00178_b200 import _lib as L
    local = dev.index
    # multi-GPU hosts: this rank's pinned buffers and its copies belong on the NUMA node of
    # its GPU's PCIe slot (best effort; -1 = unknown or a single node: nothing changed)
    saved_cpus = os.sched_getaffinity(0)
    numa_node = int(L.load().pyrit_numa_bind_thread(local))
    if wl.op == "encode":
        host_in = torch.empty((wl.k, sym), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(s0[2])
        host_out = torch.empty((wl.m, sym), dtype=torch.uint8, pin_memory=True)
        a_in, a_out = host_in.numpy(), host_out.numpy()

        def call():
            P.encode_host(a_in, wl.code, device=local, parity=a_out)
        h2d, d2h = wl.k * sym, wl.m * sym
    else:
        host = torch.empty((wl.k + wl.m, sym), dtype=torch.uint8, pin_memory=True)
        host.copy_(s0[2])
        a = host.numpy()

        def call():
            P.decode_host(a, wl.erased, wl.code, device=local)
        h2d, d2h = wl.k * sym, len(wl.erased) * sym
    for _ in range(2):
        call()
    times = []
    for _ in range(steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([statistics.mean(times)], dtype=torch.float64,
                     device=dev if os.environ.get("PYRIT_B200_DIST_BACKEND", "nccl") == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = True
    if wl.op == "encode":
        ok = bool(torch.equal(host_out.to(dev), s0[3]))
    if numa_node >= 0:
        os.sched_setaffinity(0, saved_cpus)
    return {"numa_node": numa_node, "value": wl.source_bytes() / t.item() / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": t.item() * 1e3, "steps": steps,
            "api": "pyrit_encode_host" if wl.op == "encode" else "pyrit_decode_host", "pinned": True,
            "matches_device_path": ok}


if __name__ == "__main__":
    sys.exit(main())

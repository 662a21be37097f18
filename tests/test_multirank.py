"""Multi-rank path on CPU (gloo, world_size 2 and 4): byte-offset sharding of every
strip, per-rank encode of the shard through the compiled program
(host interpreter: no GPU here), the K3 digest "checksum of checksums" gathered
across ranks, and the max-over-ranks timing reduction bench.py performs with NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_1709_00178_b200.workloads import WORKLOADS, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, strip, q):
    import torch
    import torch.distributed as dist

    import paper_1709_00178_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = WORKLOADS[5]
        w = wl.fld.w
        lo, hi = shard(strip, rank, world)
        L = hi - lo
        # this rank's shard of every fragment is itself a SymbolBuffer of w strips of L bytes
        data = [np.concatenate([O.fill_np(wl.seed, j, L, begin=s * strip + lo) for s in range(w)])
                for j in range(wl.k)]
        plan = P.Plan.encode(wl.code)
        parity = plan.interpret(data, L)
        # digest of the rank's piece of output i, with global word offsets
        dg = []
        for i in range(wl.m):
            tot = 0
            for s in range(w):
                tot += O.digest_np(parity[i][s * L:(s + 1) * L], (s * strip + lo) // 8)
            dg.append(tot % 2**64)
        t = torch.tensor([x - 2**64 if x >= 2**63 else x for x in dg], dtype=torch.int64)
        allg = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allg, t)
        ms = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if rank == 0:
            summed = [sum(int(a[i].item()) % 2**64 for a in allg) % 2**64 for i in range(wl.m)]
            q.put((summed, float(ms.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_encode_digests_match_whole(world):
    import torch.multiprocessing as mp

    wl = WORKLOADS[5]
    w = wl.fld.w
    strip = 16 * 203  # not divisible by the world size in 16-byte units
    # whole-buffer reference, computed by the oracle
    data = [O.fill_np(wl.seed, j, w * strip) for j in range(wl.k)]
    of = O.Field(w, wl.fld.n, 0, 1, w, wl.fld.modulus)
    want = O.ring_replay(of, O.cauchy(wl.k, wl.m, of), data, strip)
    whole = [O.digest_np(x, 0) for x in want]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strip, q)) for r in range(world)]
    for p in procs:
        p.start()
    summed, ms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert summed == whole
    assert ms == float(world)  # max over ranks


def test_shards_partition_every_strip():
    # column_windows analogue (test_codec.cpp:214-226): cover [0, S) exactly, 16-byte aligned cuts
    for strip in (16, 160, 44739248, 16 * 203):
        for world in (1, 2, 3, 4, 8):
            expect = 0
            for r in range(world):
                lo, hi = shard(strip, r, world)
                assert lo == expect and lo % 16 == 0
                expect = hi
            assert expect == strip

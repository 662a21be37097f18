"""Reentrancy (SPEC: concurrent calls with disjoint outputs are allowed).

Several host threads call the C ABI at the same time. Each thread has its own stream and its own
code, erasure pattern or host buffers, so plans are compiled, JIT-compiled and cached
concurrently. Every thread's result must equal the oracle's. ctypes releases the GIL for the
whole foreign call, so the library really runs concurrently.
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from tests.helpers import ofield

CODES = [
    P.CodeSpec(4, 2, P.FieldSpec.gf16_aop()),
    P.CodeSpec(6, 3, P.FieldSpec.gf64_esp()),
    P.CodeSpec(5, 3, P.FieldSpec.aop(10)),
    P.CodeSpec(7, 4, P.FieldSpec.gf256_r17()),
    P.CodeSpec(3, 5, P.FieldSpec.gf64_esp(), 1),
    P.CodeSpec(9, 2, P.FieldSpec.aop(12)),
]


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # noqa: BLE001 -- reported below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.gpu
def test_concurrent_device_encode_decode(cuda):
    import torch

    def job(idx):
        def f():
            code = CODES[idx % len(CODES)]
            w = code.field.w
            rng = np.random.default_rng(1000 + idx)
            strip = 16 * int(rng.integers(64, 1024))
            data = rng.integers(0, 256, (code.k, w * strip), dtype=np.uint8)
            want = np.stack(O.apply_columns(ofield(code.field), P.cauchy_parity_matrix(code), list(data), strip,
                                            kind=int(code.transform)))
            stream = torch.cuda.Stream(cuda)
            with torch.cuda.stream(stream):
                for rep in range(3):
                    d = torch.from_numpy(data).to(cuda, non_blocking=False)
                    parity = P.encode(d, code)
                    full = torch.cat([d, parity])
                    ref = full.clone()
                    erased = sorted(rng.choice(code.k + code.r, size=min(code.r, 1 + rep), replace=False).tolist())
                    full[erased] = 0
                    P.decode(full, erased, code)
                    stream.synchronize()
                    assert np.array_equal(parity.cpu().numpy(), want), (idx, rep)
                    assert torch.equal(full, ref), (idx, rep, erased)
        return f

    _run_threads([job(i) for i in range(12)])


@pytest.mark.gpu
def test_concurrent_host_buffer_calls(cuda):
    """pyrit_encode_host / pyrit_decode_host share one staging ring per device (serialised
    inside); concurrent callers must still each get their own correct result."""

    def job(idx):
        def f():
            code = CODES[idx % len(CODES)]
            w = code.field.w
            rng = np.random.default_rng(2000 + idx)
            ss = w * 16 * int(rng.integers(100, 1000))
            data = rng.integers(0, 256, (code.k, ss), dtype=np.uint8)
            parity = P.encode_host(data, code)
            want = np.stack(O.apply_columns(ofield(code.field), P.cauchy_parity_matrix(code), list(data), ss // w,
                                            kind=int(code.transform)))
            assert np.array_equal(parity, want), idx
            full = np.concatenate([data, parity])
            work = full.copy()
            erased = sorted(rng.choice(code.k + code.r, size=code.r, replace=False).tolist())
            work[erased] = 0
            P.decode_host(work, erased, code)
            assert np.array_equal(work, full), (idx, erased)
        return f

    _run_threads([job(i) for i in range(8)])

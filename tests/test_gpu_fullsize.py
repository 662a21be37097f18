"""BASELINE configurations at their FULL sizes on the GPU (through the C ABI).

Full-size outputs are too large for the CPU oracle to recompute in seconds, so
parity is checked through properties that do not depend on size:
  * windowed oracle: every strip's byte window [off, off+len) of the GPU output
    equals the oracle applied to the same window of the inputs (a window of an
    encode is the encode of the window -- column independence, codec.hpp:159-193),
    at the start, the middle and the end of the strips;
  * encode -> erase -> decode round trip on the GPU, compared byte for byte;
  * byte-offset shard invariance (2 and 8 shards == one launch), i.e. the
    multi-GPU split is exact;
  * the synthetic inputs themselves equal the oracle generator on those windows.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from paper_1709_00178_b200.workloads import WORKLOADS, shard

pytestmark = pytest.mark.gpu


def _ofield(f):
    return O.Field(f.w, f.n, f.kind, f.s, f.r_esp or f.w, f.modulus)


def _make(cuda, wl):
    import torch
    full = torch.empty((wl.k + wl.m, wl.frag), dtype=torch.uint8, device=cuda)
    for j in range(wl.k):
        P.fill(full[j], wl.seed, j, valid=wl.valid)
    return full


def _windows(strip, length=4096):
    mid = (strip // 2) // 16 * 16
    return [(0, length), (mid, length), (strip - length, length)]


def _check_windows(wl, full_cpu_rows, out_rows, m, strip):
    """full_cpu_rows(j, off, len) -> input window bytes (w strips x len) of symbol j."""
    f = _ofield(wl.fld)
    w = wl.fld.w
    for off, ln in _windows(strip):
        ins = [full_cpu_rows(j, off, ln) for j in range(m.shape[1])]
        want = O.ring_replay(f, m, ins, ln)
        for i, got in enumerate(out_rows(off, ln)):
            np.testing.assert_array_equal(got, want[i], err_msg=f"window {off}")
        # the generator itself, on this window of symbol 0
        if off < wl.valid // w:
            g = np.concatenate([O.fill_np(wl.seed, 0, ln, begin=s * strip + off, valid=wl.valid) for s in range(w)])
            np.testing.assert_array_equal(ins[0], g)


def _window_reader(t, strip, w):
    def read(j, off, ln):
        return np.concatenate([t[j, s * strip + off: s * strip + off + ln].cpu().numpy() for s in range(w)])
    return read


@pytest.mark.parametrize("cfg", [3, 5])
def test_full_size_encode(cuda, cfg):
    import torch
    wl = WORKLOADS[cfg]
    w, strip = wl.fld.w, wl.strip
    full = _make(cuda, wl)
    parity = P.encode(full[: wl.k], wl.code)
    full[wl.k:] = parity
    torch.cuda.synchronize()
    C = P.cauchy_parity_matrix(wl.code)
    rd = _window_reader(full, strip, w)
    _check_windows(wl, rd, lambda off, ln: [rd(wl.k + i, off, ln) for i in range(wl.m)], C, strip)

    # byte-offset shards (multi-GPU split) reproduce the single launch exactly
    plan = P.Plan.encode(wl.code)
    stream = torch.cuda.current_stream().cuda_stream
    for world in (2, 8):
        out = torch.zeros_like(parity)
        for rank in range(world):
            lo, hi = shard(strip, rank, world)
            plan.apply([full[j].data_ptr() for j in range(wl.k)], [out[i].data_ptr() for i in range(wl.m)], strip,
                       lo, hi - lo, stream=stream)
        torch.cuda.synchronize()
        assert torch.equal(out, parity), world
        del out

    # encode -> erase (data and parity) -> decode round trip
    erased = [0, 5, wl.k - 1, wl.k + 1]
    saved = full[erased].clone()
    full[erased] = 0xA5
    P.decode(full, erased, wl.code)
    torch.cuda.synchronize()
    assert torch.equal(full[erased], saved)
    del full, parity, saved
    torch.cuda.empty_cache()


def test_full_size_config4_decode(cuda):
    import torch
    wl = WORKLOADS[4]
    w, strip = wl.fld.w, wl.strip
    full = _make(cuda, wl)
    full[wl.k:] = P.encode(full[: wl.k], wl.code)
    torch.cuda.synchronize()
    rd = _window_reader(full, strip, w)
    C = P.cauchy_parity_matrix(wl.code)
    _check_windows(wl, rd, lambda off, ln: [rd(wl.k + i, off, ln) for i in range(wl.m)], C, strip)
    saved = full.clone()
    erased = list(wl.erased)
    full[erased] = 0
    P.decode(full, erased, wl.code)
    torch.cuda.synchronize()
    assert torch.equal(full, saved)
    # the repair rows themselves against the oracle on windows (fused rows over survivors)
    surv, outs, m = P.repair_matrix(wl.code, erased)
    rd2 = _window_reader(full, strip, w)
    f = _ofield(wl.fld)
    for off, ln in _windows(strip):
        ins = [rd2(int(s), off, ln) for s in surv]
        want = O.ring_replay(f, m, ins, ln)
        for i, o in enumerate(outs):
            np.testing.assert_array_equal(rd2(int(o), off, ln), want[i])
    del full, saved
    torch.cuda.empty_cache()

"""The replay operator over explicit schedules (codec.hpp:118-193): any XorSchedule --
the reference's compile_schedule / compile_crs_schedule output or hand-built op lists --
compiled by pyrit_plan_from_schedule into one fused kernel.

Checked against the oracle's op-by-op restatement of replay (oracle.replay_ops), which is
itself pinned to the reference's parallel_replay (oracle/_ref) and whose schedules are
pinned op for op to the reference's compile_schedule.  Mirrors test_schedule.cpp:32-157
(identity / zero entries, stale outputs, trimming, replay == field oracle).

CPU tests run the compiled program through the host interpreter; `gpu` tests run the
generated kernels through pyrit_cu_apply (device buffers) and pyrit_apply_host (host
buffers)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from tests.helpers import G16, G64, G256, G1024, G4096, ofield

REF = O.ref_available()


def sched_ops(f, m, kind=0, which="sparse") -> np.ndarray:
    of = ofield(f)
    if which == "crs":
        return O.compile_crs_schedule(of, m)
    return O.compile_schedule(of, m, kind, 1 if which == "dense" else 0)


def labels_of(ins, outs):
    addr = [a.ctypes.data for a in ins] + [a.ctypes.data for a in outs]
    return [addr.index(a) for a in addr]


def run_interp(f, k, outputs, ops, ins, outs, strip, off=0, length=None):
    plan = P.Plan.from_schedule(P.XorSchedule(f, k, outputs, ops), labels_of(ins, outs))
    plan.interpret(ins, strip, off, length, outs=outs)
    return plan


def random_ops(rng, f, k, outputs, count, read_outputs=True):
    """A random op list in the reference's slot conventions: destinations are output slots
    (any packet < n) or input scratch packets (>= w); sources anything in range."""
    ops = np.zeros(count, dtype=P.OP_DTYPE)
    slots = k + outputs
    for q in range(count):
        if rng.random() < 0.2:
            ds, dp = int(rng.integers(0, slots)), int(rng.integers(f.w, f.n))  # scratch of any slot
        else:
            ds, dp = int(rng.integers(k, slots)), int(rng.integers(0, f.n))
        if read_outputs:
            ss = int(rng.integers(0, slots))
        else:
            ss = int(rng.integers(0, k))
        sp = int(rng.integers(0, f.n))
        mode = int(rng.choice([0, 1, 1, 1, 2]))
        ops[q] = (ss, sp, ds, dp, mode)
    return ops


# ----------------------------------------------------------------- oracle pins
@pytest.mark.skipif(not REF, reason="reference tree not available")
@pytest.mark.parametrize("f", [G16, G64, G1024, G4096])
def test_oracle_schedules_equal_reference_op_lists(f):
    """or_compile_schedule / or_compile_crs_schedule emit the reference's op lists exactly.  (R_{2,17}
    is left out: there the reference's uint16 RingElem truncates representatives, the documented
    widening.)"""
    of = ofield(f)
    for k, r in ((1, 1), (3, 2), (2, 5), (5, 5)):
        if k + r > (1 << f.w):
            continue
        m = O.cauchy(k, r, of)
        for kind in (0, 1):
            for rep in (0, 1):
                assert np.array_equal(O.compile_schedule(of, m, kind, rep), O.ref_schedule_ops(of, m, kind, 0, rep))
        assert np.array_equal(O.compile_crs_schedule(of, m), O.ref_schedule_ops(of, m, 0, 1))


@pytest.mark.skipif(not REF, reason="reference tree not available")
def test_oracle_replay_equals_reference_replay():
    """or_replay_ops == the reference's parallel_replay on random schedules, separate buffers and
    decode()-style in place (one SymbolBuffer, in and out maps into it)."""
    rng = np.random.default_rng(11)
    for f in (G16, G64):
        of = ofield(f)
        for trial in range(12):
            k, outputs = int(rng.integers(1, 5)), int(rng.integers(1, 4))
            ss = f.w * 8 * int(rng.integers(1, 5))
            strip = ss // f.w
            ops = random_ops(rng, f, k, outputs, int(rng.integers(1, 40)))
            ops = ops[~((ops["dst_sym"] < k) & (ops["dst_pkt"] < f.w))]
            nin = k + 2
            inp = rng.integers(0, 256, (nin, ss), dtype=np.uint8)
            out = rng.integers(0, 256, (outputs + 1, ss), dtype=np.uint8)
            in_map = rng.permutation(nin)[:k]
            out_map = rng.permutation(outputs + 1)[:outputs]
            want = out.copy()
            O.ref_replay_ops(of, k, outputs, ops, inp, in_map, want, out_map, ss, threads=1 + trial % 3)
            got = out.copy()
            O.replay_ops(of, k, outputs, ops, [inp[j] for j in in_map], [got[i] for i in out_map], strip)
            assert np.array_equal(got, want)
            # in place: one buffer, disjoint maps (decode passes survivors / erased)
            buf = rng.integers(0, 256, (k + outputs, ss), dtype=np.uint8)
            perm = rng.permutation(k + outputs)
            im, om = perm[:k], perm[k:]
            want = buf.copy()
            O.ref_replay_ops(of, k, outputs, ops, None, im, want, om, ss)
            got = buf.copy()
            O.replay_ops(of, k, outputs, ops, [got[j] for j in im], [got[i] for i in om], strip)
            assert np.array_equal(got, want)


# ------------------------------------------------------- compiled schedules (CPU)
@pytest.mark.parametrize("f", [G16, G64])
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("which", ["sparse", "dense", "crs"])
def test_reference_schedules_compile_to_replay(f, kind, which):
    """test_schedule.cpp:104-136 on the operator: every (k, r) <= 5, the reference's schedule
    compiled for the GPU == op-by-op replay, with slot maps and stale outputs."""
    if which == "crs" and kind == 1:
        pytest.skip("CRS schedules are plain field codes")
    rng = np.random.default_rng(f.w * 10 + kind)
    of = ofield(f)
    for k in range(1, 6):
        for r in range(1, 6):
            m = O.cauchy(k, r, of)
            ops = sched_ops(f, m, kind, which)
            ss = f.w * 8 * 3
            strip = ss // f.w
            inp = rng.integers(0, 256, (k + 1, ss), dtype=np.uint8)
            in_map = rng.permutation(k + 1)[:k]
            stale = rng.integers(0, 256, (r, ss), dtype=np.uint8)
            want = stale.copy()
            O.replay_ops(of, k, r, ops, [inp[j] for j in in_map], [want[i] for i in range(r)], strip)
            got = stale.copy()
            plan = run_interp(f, k, r, ops, [inp[j] for j in in_map], [got[i] for i in range(r)], strip)
            assert np.array_equal(got, want), (k, r)
            # and == the field oracle (the schedule is a plain GF(2^w) code)
            field = np.stack(O.apply_columns(of, m, [inp[j] for j in in_map], strip, kind=kind))
            assert np.array_equal(got, field)
            assert plan.stats()["ref_region_ops"] == len(ops)


def test_identity_and_zero_entries():
    """test_schedule.cpp:32-80: [1] -> w Copies + w post XORs reading scratch; [0] -> w explicit
    Zero ops, and a stale output is cleared."""
    f = G16
    of = ofield(f)
    ss = 4 * 16
    rng = np.random.default_rng(3)
    d = rng.integers(0, 256, (1, ss), dtype=np.uint8)
    ops1 = sched_ops(f, np.array([[1]], dtype=np.uint16))
    assert list(ops1["mode"][: f.w]) == [0] * f.w and (ops1["src_pkt"][f.w:] >= f.w).all()
    out = rng.integers(0, 256, (1, ss), dtype=np.uint8)
    run_interp(f, 1, 1, ops1, [d[0]], [out[0]], ss // f.w)
    assert np.array_equal(out, d)
    ops0 = sched_ops(f, np.array([[0]], dtype=np.uint16))
    assert len(ops0) == f.w + f.w and (ops0["mode"][: f.w] == 2).all()
    out = rng.integers(0, 256, (1, ss), dtype=np.uint8)
    run_interp(f, 1, 1, ops0, [d[0]], [out[0]], ss // f.w)
    assert not out.any()


@pytest.mark.parametrize("f", [G16, G64, G256])
def test_random_schedules(f):
    """Hand-built op lists: outputs read before they are written (prior contents), scratch read
    before it is written (zero), Zero ops, partly written outputs (untouched strips), slot maps,
    column windows."""
    rng = np.random.default_rng(f.n)
    of = ofield(f)
    for trial in range(40):
        k, outputs = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        ops = random_ops(rng, f, k, outputs, int(rng.integers(0, 30)))
        ops = ops[~((ops["dst_sym"] < k) & (ops["dst_pkt"] < f.w))]
        ss = f.w * 8 * int(rng.integers(1, 6))
        strip = ss // f.w
        off = int(rng.integers(0, strip))
        length = int(rng.integers(0, strip - off + 1))
        inp = rng.integers(0, 256, (k, ss), dtype=np.uint8)
        out0 = rng.integers(0, 256, (outputs, ss), dtype=np.uint8)
        want = out0.copy()
        O.replay_ops(of, k, outputs, ops, list(inp), list(want), strip, off, length)
        got = out0.copy()
        run_interp(f, k, outputs, ops, list(inp), list(got), strip, off, length)
        assert np.array_equal(got, want), trial


@pytest.mark.parametrize("f", [G16, G64])
def test_shared_storage(f):
    """Slots that name the same symbol share storage (decode() replays one SymbolBuffer as in
    and out): in place with overlapping maps, and two output slots on one symbol."""
    rng = np.random.default_rng(99 + f.w)
    of = ofield(f)
    for trial in range(40):
        k, outputs = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        nsym = int(rng.integers(max(k, outputs), k + outputs + 1))
        ops = random_ops(rng, f, k, outputs, int(rng.integers(1, 30)))
        ops = ops[~((ops["dst_sym"] < k) & (ops["dst_pkt"] < f.w))]
        ss = f.w * 8 * 2
        strip = ss // f.w
        buf = rng.integers(0, 256, (nsym, ss), dtype=np.uint8)
        im = rng.integers(0, nsym, k)
        om = rng.integers(0, nsym, outputs)
        want = buf.copy()
        O.replay_ops(of, k, outputs, ops, [want[j] for j in im], [want[i] for i in om], strip)
        got = buf.copy()
        run_interp(f, k, outputs, ops, [got[j] for j in im], [got[i] for i in om], strip)
        assert np.array_equal(got, want), trial


def test_schedule_errors():
    """replay's errors (codec.hpp:122-143): writing an input data packet and slots/packets out of
    range are BufferShape; no work is done."""
    f = G16
    bad = np.array([(0, 0, 0, 1, 0)], dtype=P.OP_DTYPE)  # Copy into input slot 0, packet 1
    with pytest.raises(P.PyritError) as e:
        P.Plan.from_schedule(P.XorSchedule(f, 1, 1, bad))
    assert e.value.code == "BufferShape"
    for op in [(0, 0, 2, 0, 0), (0, 5, 1, 0, 1), (3, 0, 1, 0, 1), (0, 0, 1, 0, 3)]:
        with pytest.raises(P.PyritError):
            P.Plan.from_schedule(P.XorSchedule(f, 1, 1, np.array([op], dtype=P.OP_DTYPE)))
    # scratch of an input slot is writable (Parity pre phase)
    ok = np.array([(0, 0, 0, 4, 0), (0, 4, 1, 0, 0)], dtype=P.OP_DTYPE)
    P.Plan.from_schedule(P.XorSchedule(f, 1, 1, ok))
    # an empty schedule writes nothing
    plan = P.Plan.from_schedule(P.XorSchedule(f, 2, 1, np.zeros(0, dtype=P.OP_DTYPE)))
    a = np.arange(32, dtype=np.uint8)
    o = np.full(32, 7, dtype=np.uint8)
    plan.interpret([a, a], 8, outs=[o])
    assert (o == 7).all()


def test_field_schedules_compile_to_the_ring_program():
    """Matrix recovery: a schedule whose map is a GF(2^w) matrix (every compile_schedule /
    compile_crs_schedule output for AOP/ESP fields, ring, dense or CRS) compiles to the same ring
    program as the matrix itself -- same tuning key, same kernel -- so replaying the reference's
    schedule costs what encode() costs.  R_{2,17} ring schedules from the reference are not field
    maps (uint16 truncation): they replay as their own bit map, bytes as the reference's."""
    from paper_1709_00178_b200.workloads import WORKLOADS
    for c in (1, 3, 5):
        wl = WORKLOADS[c]
        of = ofield(wl.fld)
        m = P.cauchy_parity_matrix(wl.code)
        enc = P.Plan.encode(wl.code)
        for ops in (O.compile_schedule(of, m), O.compile_crs_schedule(of, m), O.compile_schedule(of, m, 0, 1)):
            p = P.Plan.from_schedule(P.XorSchedule(wl.fld, wl.k, wl.m, ops))
            assert p.key() == enc.key()
            assert p.source(P._lib.SOURCE_STAGED)[0] == enc.source(P._lib.SOURCE_STAGED)[0]
            assert p.stats()["ref_region_ops"] == len(ops)
    wl = WORKLOADS[2]
    of = ofield(wl.fld)
    m = P.cauchy_parity_matrix(wl.code)
    crs = P.Plan.from_schedule(P.XorSchedule(wl.fld, wl.k, wl.m, O.compile_crs_schedule(of, m)))
    assert crs.key() == P.Plan.encode(wl.code).key()
    ring = P.Plan.from_schedule(P.XorSchedule(wl.fld, wl.k, wl.m, O.compile_schedule(of, m)))
    assert "sch" in ring.key()


def test_c_abi_argument_errors():
    """pyrit_plan_from_schedule / pyrit_apply_host validate their arguments before any device work
    (return codes are 1 + Errc, errors.hpp:12-24)."""
    import ctypes as C
    from paper_1709_00178_b200 import _lib as L
    lib = L.load()
    f = G16.c()
    h = C.c_void_p()
    assert lib.pyrit_plan_from_schedule(C.byref(f), 1, 1, None, 3, None, C.byref(h)) == 11  # InvalidArgument
    assert lib.pyrit_plan_from_schedule(C.byref(f), 0, 1, None, 0, None, C.byref(h)) == 11  # no input slots
    ops = np.array([(0, 0, 1, 0, 0)], dtype=P.OP_DTYPE)
    plan = P.Plan.from_schedule(P.XorSchedule(G16, 1, 1, ops))
    a = np.zeros(64, dtype=np.uint8)
    arr = (C.c_void_p * 1)(a.ctypes.data)
    assert lib.pyrit_apply_host(plan._h, None, arr, 16, 0, 16, 0) == 11
    assert lib.pyrit_apply_host(plan._h, arr, arr, 16, 8, 16, 0) == 4  # BufferShape: window past the strip
    nul = (C.c_void_p * 1)(None)
    assert lib.pyrit_apply_host(plan._h, nul, arr, 16, 0, 16, 0) == 11  # null symbol pointer


# ------------------------------------------------------------------------- GPU
def _torch():
    import torch
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("f", [G16, G64, G256, G1024, G4096])
def test_gpu_reference_schedules(cuda, f):
    """The reference's own schedules (sparse/dense ring, both transforms, CRS) replayed on the GPU
    through P.replay == op-by-op replay; sizes that take the staged and the direct kernel."""
    torch = _torch()
    of = ofield(f)
    rng = np.random.default_rng(f.w)
    codes = [(4, 2), (10, 4), (16, 4)] if f.w >= 8 else [(4, 2), (3, 5), (8, 4)]
    for k, r in codes:
        if k + r > (1 << f.w):
            continue
        m = O.cauchy(k, r, of)
        for kind, which in ((0, "sparse"), (0, "dense"), (0, "crs"), (1, "sparse")):
            ops = sched_ops(f, m, kind, which)
            sched = P.XorSchedule(f, k, r, ops)
            for strip in (16 * 1000, 4104, 2 * 777):
                ss = f.w * strip
                inp = rng.integers(0, 256, (k + 1, ss), dtype=np.uint8)
                out0 = rng.integers(0, 256, (r, ss), dtype=np.uint8)
                in_map = list(rng.permutation(k + 1)[:k])
                out_map = list(range(r))
                want = out0.copy()
                O.replay_ops(of, k, r, ops, [inp[j] for j in in_map], list(want), strip)
                di = torch.from_numpy(inp).to(cuda)
                do = torch.from_numpy(out0).to(cuda)
                P.replay(sched, di, in_map, do, out_map)
                torch.cuda.synchronize()
                assert np.array_equal(do.cpu().numpy(), want), (k, r, kind, which, strip)
                assert P.Plan.last_launch()["kernel"].startswith("pyrit_ring_")
                got = out0.copy()
                P.replay(sched, inp, in_map, got, out_map)  # host buffers
                assert np.array_equal(got, want), (k, r, kind, which, strip, "host")


@pytest.mark.gpu
def test_gpu_replay_of_baseline_schedule_uses_the_encode_kernel(cuda):
    """The reference's compile_schedule output for BASELINE config 5 (strip shrunk), replayed through
    P.replay, launches the same generated kernel as encode() and gives the same parity."""
    torch = _torch()
    from paper_1709_00178_b200.workloads import WORKLOADS
    wl = WORKLOADS[5]
    of = ofield(wl.fld)
    m = P.cauchy_parity_matrix(wl.code)
    strip = 16 * 65536
    data = torch.from_numpy(np.random.default_rng(5).integers(0, 256, (wl.k, wl.fld.w * strip),
                                                               dtype=np.uint8)).to(cuda)
    parity = P.encode(data, wl.code)
    torch.cuda.synchronize()
    enc_kernel = P.Plan.last_launch()["kernel"]
    out = torch.zeros_like(parity)
    P.parallel_replay(P.XorSchedule(wl.fld, wl.k, wl.m, O.compile_schedule(of, m)), data, list(range(wl.k)), out,
                      list(range(wl.m)))
    torch.cuda.synchronize()
    assert P.Plan.last_launch()["kernel"] == enc_kernel
    assert torch.equal(out, parity)


@pytest.mark.gpu
@pytest.mark.parametrize("f", [G16, G64, G256])
def test_gpu_random_and_in_place_schedules(cuda, f):
    """Hand-built schedules on the GPU: prior output contents, zero scratch, partly written outputs,
    column windows, and in-place replay in one buffer (overlapping maps) -- device and host paths."""
    torch = _torch()
    of = ofield(f)
    rng = np.random.default_rng(200 + f.w)
    for trial in range(24):
        k, outputs = int(rng.integers(1, 6)), int(rng.integers(1, 4))
        ops = random_ops(rng, f, k, outputs, int(rng.integers(1, 40)))
        ops = ops[~((ops["dst_sym"] < k) & (ops["dst_pkt"] < f.w))]
        sched = P.XorSchedule(f, k, outputs, ops)
        strip = [16 * 4096, 4 * 999, 16 * 64 + 8][trial % 3]
        ss = f.w * strip
        nsym = k + outputs
        buf = rng.integers(0, 256, (nsym, ss), dtype=np.uint8)
        if trial % 2:
            im, om = list(rng.integers(0, nsym, k)), list(rng.integers(0, nsym, outputs))  # shared storage
        else:
            perm = rng.permutation(nsym)
            im, om = list(perm[:k]), list(perm[k:])
        off = int(rng.integers(0, 64)) * 4 if trial % 4 == 3 else 0
        length = strip - off - (int(rng.integers(0, 16)) * 4 if trial % 4 == 3 else 0)
        want = buf.copy()
        O.replay_ops(of, k, outputs, ops, [want[j] for j in im], [want[i] for i in om], strip, off, length)
        d = torch.from_numpy(buf).to(cuda)
        P.replay(sched, d, im, d, om, off, length)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), want), trial
        got = buf.copy()
        P.replay(sched, got, im, got, om, off, length)
        assert np.array_equal(got, want), (trial, "host")

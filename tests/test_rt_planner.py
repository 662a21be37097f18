"""CPU check of the runtime-matrix ring kernel's launch planner (csrc/runtime.cpp build_ring_rt).

`pyrit_rt_interpret` runs, on host buffers, exactly the plan a ring_rt launch
would get -- output groups and parts (heaviest output onto the lightest bin),
the op lists read back from the kernel parameters, sentinels, the parity
extension, the fold, column windows, stripe batches, and the op budget that
splits a code over several launches -- so these tests hold the planner
bit-exact against the oracle (oracle/, pinned to the reference in
test_oracle.py) without a GPU.  The GPU runs of the same plans are in
test_gpu_ring_rt.py.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1709_00178_b200 as P
from paper_1709_00178_b200.workloads import WORKLOADS
from tests.helpers import G16, G64, G256, G1024, G4096, oracle_ring, rand_symbols

FIELDS = [G16, G64, G256, G1024, G4096]


def aligned(shape, fill=None) -> np.ndarray:
    """A C-contiguous uint8 array whose rows start on 64-byte boundaries."""
    rows, cols = shape
    raw = np.zeros(rows * cols + 64, dtype=np.uint8)
    start = (-raw.ctypes.data) % 64
    a = raw[start:start + rows * cols].reshape(rows, cols)
    assert a.ctypes.data % 64 == 0 and cols % 16 == 0
    if fill is not None:
        a[...] = fill
    return a


def run_rt(plan, data: np.ndarray, rows: int, strip: int, off=0, length=None, stripes=1) -> np.ndarray:
    out = aligned((stripes * rows, data.shape[1]), 0x5A)
    if stripes == 1:
        plan.interpret_rt([data[j].ctypes.data for j in range(data.shape[0])],
                          [out[i].ctypes.data for i in range(rows)], strip, off, length)
    else:  # stripe b of input j at data[b*k + j]: pitch = k symbols; outputs likewise
        k = data.shape[0] // stripes
        sym = data.shape[1]
        plan.interpret_rt([data[j].ctypes.data for j in range(k)], [out[i].ctypes.data for i in range(rows)], strip,
                          off, length, stripes, k * sym, rows * sym)
    return out


@pytest.mark.parametrize("f", FIELDS, ids=lambda f: f"w{f.w}n{f.n}")
@pytest.mark.parametrize("kind", [0, 1])
def test_planner_random_matrices(f, kind):
    """e = 1 .. past one launch (1, 2 and 4 parts, idle parts, output groups, further
    launches), k up to 64, zero entries."""
    rng = np.random.default_rng(77 * f.w + kind)
    for e, k in [(1, 1), (2, 3), (3, 7), (4, 10), (5, 16), (8, 12), (9, 5), (17, 3), (4, 64), (20, 40), (40, 3)]:
        m = rng.integers(0, 1 << f.w, (e, k), dtype=np.uint16)
        m[rng.random((e, k)) < 0.1] = 0
        plan = P.Plan.create(f, m, P.TransformKind(kind))
        strip = 2048 + 32 * f.w  # one full 2 KiB tile and part of a second
        data = aligned((k, f.w * strip))
        data[...] = rand_symbols(k, f.w * strip, int(rng.integers(1 << 30)))
        got = run_rt(plan, data, e, strip)
        np.testing.assert_array_equal(got, oracle_ring(f, m, data, kind=kind), err_msg=f"e={e} k={k}")
        plan.close()


def test_planner_op_budget_splits_launches():
    """A (100 x 64) matrix over GF(2^4)/R_{2,5}: its 100 outputs fit one launch's output
    groups (8 groups x 16), but its ring terms exceed one launch's op budget (8192
    bytes), so the planner splits the outputs over launches instead of failing."""
    f = G16
    rng = np.random.default_rng(5)
    m = rng.integers(1, 1 << f.w, (100, 64), dtype=np.uint16)
    plan = P.Plan.create(f, m)
    terms = sum(bin(int(r)).count("1") for r in plan.reps().ravel())
    assert terms > 8192
    strip = 2048
    data = aligned((64, f.w * strip))
    data[...] = rand_symbols(64, f.w * strip, 9)
    np.testing.assert_array_equal(run_rt(plan, data, 100, strip), oracle_ring(f, m, data))


@pytest.mark.parametrize("f", [G256, G4096], ids=lambda f: f"w{f.w}n{f.n}")
def test_planner_windows_and_batches(f):
    rng = np.random.default_rng(11)
    k, e = 6, 3
    m = rng.integers(1, 1 << f.w, (e, k), dtype=np.uint16)
    plan = P.Plan.create(f, m)
    strip = 4096 + 48
    data = aligned((k, f.w * strip))
    data[...] = rand_symbols(k, f.w * strip, 3)
    want = oracle_ring(f, m, data)
    off, length = 2048 + 16, 1024 + 32
    got = run_rt(plan, data, e, strip, off, length)
    for i in range(e):
        for s in range(f.w):
            a, b = s * strip + off, s * strip + off + length
            np.testing.assert_array_equal(got[i, a:b], want[i, a:b])
            assert (got[i, s * strip:a] == 0x5A).all() and (got[i, b:(s + 1) * strip] == 0x5A).all()
    # stripe batch: 3 stripes, input j of stripe b at data[b*k + j]
    nb = 3
    batch = aligned((nb * k, f.w * strip))
    batch[...] = rand_symbols(nb * k, f.w * strip, 4)
    got = run_rt(plan, batch, e, strip, stripes=nb)
    for b in range(nb):
        np.testing.assert_array_equal(got[b * e:(b + 1) * e], oracle_ring(f, m, batch[b * k:(b + 1) * k]))


@pytest.mark.parametrize("erased", [(1, 6, 9, 10), (0, 1, 2, 3), (3, 11), (13,), (4, 5, 12, 13)])
def test_planner_config4_decode_rows(erased):
    """The fused repair rows of config-4 erasure patterns (survivor-inverse rows, parity
    rows composed on the host) planned for the runtime kernel repair the symbols."""
    wl = WORKLOADS[4]
    f = wl.fld
    strip = 2048
    data = aligned((wl.k, f.w * strip))
    data[...] = rand_symbols(wl.k, f.w * strip, 21)
    full = np.concatenate([data, oracle_ring(f, P.cauchy_parity_matrix(wl.code), data)])
    plan = P.Plan.decode(wl.code, erased)
    ins = aligned((wl.k, f.w * strip))
    ins[...] = full[list(plan.survivors)]
    got = run_rt(plan, ins, len(plan.outputs), strip)
    np.testing.assert_array_equal(got, full[list(plan.outputs)])


def test_planner_rejects_ineligible_launches():
    f = G256
    m = np.ones((2, 3), dtype=np.uint16)
    plan = P.Plan.create(f, m)
    data = aligned((3, f.w * 2048))
    out = aligned((2, f.w * 2048))
    with pytest.raises(P.PyritError):  # 8-byte misaligned input
        plan.interpret_rt([data[0].ctypes.data + 8, data[1].ctypes.data, data[2].ctypes.data],
                          [out[0].ctypes.data, out[1].ctypes.data], 2048)
    with pytest.raises(P.PyritError):  # window out of range
        plan.interpret_rt([data[j].ctypes.data for j in range(3)], [out[i].ctypes.data for i in range(2)], 2048,
                          1024, 2048)


@pytest.mark.parametrize("f", [G256, G4096], ids=lambda f: f"w{f.w}n{f.n}")
def test_planner_negative_control(f):
    """The check can fail: one flipped bit of one representative (pyrit_plan_inject_fault,
    cf. the reference's --inject-theta-fault, selfcheck.hpp:28-34) changes exactly the
    output row it belongs to."""
    rng = np.random.default_rng(3)
    k, e = 10, 4
    m = rng.integers(1, 1 << f.w, (e, k), dtype=np.uint16)
    plan = P.Plan.create(f, m)
    strip = 2048
    data = aligned((k, f.w * strip))
    data[...] = rand_symbols(k, f.w * strip, 8)
    want = oracle_ring(f, m, data)
    np.testing.assert_array_equal(run_rt(plan, data, e, strip), want)
    plan.inject_fault(2 * k + 3, 1)  # entry (2, 3)
    bad = run_rt(plan, data, e, strip)
    assert not np.array_equal(bad[2], want[2])
    for i in (0, 1, 3):
        np.testing.assert_array_equal(bad[i], want[i])


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@st.composite
def rt_cases(draw):
    f = draw(st.sampled_from(FIELDS))
    kind = draw(st.sampled_from([0, 0, 1]))
    e = draw(st.integers(1, 40))
    k = draw(st.integers(1, 64))
    strip = 16 * draw(st.integers(1, 400))
    off = 16 * draw(st.integers(0, strip // 16 - 1))
    length = 16 * draw(st.integers(1, (strip - off) // 16))
    nb = draw(st.sampled_from([1, 1, 2, 3]))
    seed = draw(st.integers(0, 2**31 - 1))
    return f, kind, e, k, strip, off, length, nb, seed


@settings(max_examples=120, deadline=None)
@given(rt_cases())
def test_planner_property(case):
    """Random geometry, transform, output count (parts, groups, launches), input count,
    strip, column window and stripe batch: the runtime-matrix launch plan reproduces the
    oracle inside the window and leaves every byte outside it untouched."""
    f, kind, e, k, strip, off, length, nb, seed = case
    rng = np.random.default_rng(seed)
    m = rng.integers(0, 1 << f.w, (e, k), dtype=np.uint16)
    plan = P.Plan.create(f, m, P.TransformKind(kind))
    sym = f.w * strip
    data = aligned((nb * k, sym))
    data[...] = rng.integers(0, 256, (nb * k, sym), dtype=np.uint8)
    got = run_rt(plan, data, e, strip, off, length, stripes=nb)
    for b in range(nb):
        want = oracle_ring(f, m, data[b * k:(b + 1) * k], kind=kind)
        for i in range(e):
            for s in range(f.w):
                lo, hi = s * strip + off, s * strip + off + length
                row = got[b * e + i]
                np.testing.assert_array_equal(row[lo:hi], want[i, lo:hi])
                assert (row[s * strip:lo] == 0x5A).all() and (row[hi:(s + 1) * strip] == 0x5A).all()
    plan.close()


def _poly_mod(a: int, p: int) -> int:
    dp = p.bit_length() - 1
    while a and a.bit_length() - 1 >= dp:
        a ^= p << (a.bit_length() - 1 - dp)
    return a


def _clmul(a: int, b: int) -> int:
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        b >>= 1
    return r


@pytest.mark.parametrize("f", FIELDS, ids=lambda f: f"w{f.w}n{f.n}")
@pytest.mark.parametrize("kind", [0, 1])
def test_ringmat_any_representative(f, kind):
    """pyrit_plan_from_ringmat (SURVEY 8(b)'s ring-matrix operand): raw n-bit masks, minimal or
    not -- every element u of a coset stands for the field element u mod p -- give the
    oracle's symbols for the field matrix, both on the runtime kernel's plan (the masks as
    given) and through the compiled program (the field matrix)."""
    rng = np.random.default_rng(13 * f.w + kind)
    e, k = 5, 9
    m = rng.integers(0, 1 << f.w, (e, k), dtype=np.uint16)
    reps = np.zeros((e, k), dtype=np.uint32)
    for i in range(e):
        for j in range(k):
            u = P.sparse_transform(int(m[i, j]), f)
            # Embedding: any element of the coset; Parity: the canonical one
            t = int(rng.integers(0, 1 << (f.n - f.w))) if kind == 0 else 0
            reps[i, j] = u ^ _clmul(t, f.modulus)  # another element of the same coset
            assert reps[i, j] < (1 << f.n) and _poly_mod(int(reps[i, j]), f.modulus) == m[i, j]
    plan = P.Plan.from_ringmat(f, reps, P.TransformKind(kind))
    np.testing.assert_array_equal(plan.reps(), reps)
    strip = 2048 + 16 * f.w
    data = aligned((k, f.w * strip))
    data[...] = rand_symbols(k, f.w * strip, 31)
    want = oracle_ring(f, m, data, kind=kind)
    np.testing.assert_array_equal(run_rt(plan, data, e, strip), want)
    got = np.stack(plan.interpret([data[j] for j in range(k)], strip))  # the compiled program
    np.testing.assert_array_equal(got, want)


def test_ringmat_rejects_wide_elements():
    f = G256
    with pytest.raises(P.PyritError):
        P.Plan.from_ringmat(f, np.array([[1 << 17]], dtype=np.uint32))
    u = P.sparse_transform(7, f)
    P.Plan.from_ringmat(f, np.array([[u ^ f.modulus]], dtype=np.uint32))  # Embedding: any coset element
    with pytest.raises(P.PyritError):  # Parity: only the canonical representative
        P.Plan.from_ringmat(f, np.array([[u ^ f.modulus]], dtype=np.uint32), P.TransformKind.Parity)
    with pytest.raises(P.PyritError):
        P.Plan.from_ringmat(f, np.zeros((0, 3), dtype=np.uint32))


def test_planner_pairs_shifts_within_the_case_budget():
    """Paired-shift cases (runtime.cpp rt_select_pairs): a four-output plan runs fewer ops
    than its matrix has ring terms (a pair op covers two shifts of one representative),
    the dispatch-case code the ops name stays within the instruction-cache budget, and a
    single-output plan (V = 2 instance, no pair cases) runs one op per term."""
    for c in (2, 3, 4, 5):
        wl = WORKLOADS[c]
        plan = P.Plan.decode(wl.code, list(wl.erased)) if wl.op == "decode" else P.Plan.encode(wl.code)
        info = plan.rt_info()
        assert info["launches"] == 1
        assert info["terms"] // 2 <= info["ops"] < info["terms"], info
        assert 0 < info["case_bytes"] <= 26 * 1024, info
    wl = WORKLOADS[4]
    one = P.Plan.decode(wl.code, [3]).rt_info()
    assert one["ops"] == one["terms"]

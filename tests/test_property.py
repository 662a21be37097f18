"""Property tests of the ring program compiler on CPU (hypothesis), beyond the reference's two
fields. The embedding path is valid for ANY modulus p dividing x^n + 1: a representative only has
to be congruent to the entry mod p (ring.hpp:77-90), and the fold x^t mod p generalises
transform.hpp:39-46. So random matrices over GF(2^w) embedded in R_{2,n}, for several (w, n, p),
must give the plain field code (the oracle's column-at-a-time oracle_apply, codec.hpp:444-469).
The compiled program runs through its host interpreter; the sizes and windows are random.
"""
from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O
import paper_1709_00178_b200 as P
from tests.helpers import ofield

# (w, n, p): p irreducible of degree w dividing x^n + 1
FIELDS = [
    P.FieldSpec(2, 3, 0, 1, 2, 0b111),
    P.FieldSpec(3, 7, 0, 1, 3, 0b1011),
    P.FieldSpec(3, 7, 0, 1, 3, 0b1101),
    P.FieldSpec(4, 15, 0, 1, 4, 0b10011),
    P.FieldSpec.gf16_aop(),
    P.FieldSpec.gf64_esp(),
    P.FieldSpec.gf256_r17(),
    P.FieldSpec.aop(10),
    P.FieldSpec.aop(12),
]


@st.composite
def cases(draw):
    f = draw(st.sampled_from(FIELDS))
    k = draw(st.integers(1, 6))
    r = draw(st.integers(1, 5))
    entries = draw(st.lists(st.integers(0, (1 << f.w) - 1), min_size=k * r, max_size=k * r))
    m = np.array(entries, dtype=np.uint16).reshape(r, k)
    strip = draw(st.integers(1, 40))
    off = draw(st.integers(0, strip - 1))
    length = draw(st.integers(1, strip - off))
    rep = draw(st.sampled_from([P.RingRep.Sparse, P.RingRep.Dense, 2]))
    seed = draw(st.integers(0, 2**31))
    return f, m, strip, off, length, rep, seed


@settings(max_examples=400, deadline=None)
@given(cases())
def test_random_matrices_any_field(case):
    f, m, strip, off, length, rep, seed = case
    rng = np.random.default_rng(seed)
    r, k = m.shape
    ins = [rng.integers(0, 256, f.w * strip, dtype=np.uint8) for _ in range(k)]
    want = O.apply_columns(ofield(f), m, ins, strip, off=off, length=length,
                           outs=[np.full(f.w * strip, 0x5A, dtype=np.uint8) for _ in range(r)])
    plan = P.Plan.create(f, m, rep=rep)
    got = plan.interpret(ins, strip, off, length, outs=[np.full(f.w * strip, 0x5A, dtype=np.uint8) for _ in range(r)])
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("f", FIELDS, ids=lambda f: f"w{f.w}n{f.n}p{f.modulus:x}")
def test_representatives_any_field(f):
    """rep = sparse_transform(u) is congruent to u mod p and has the least weight in its coset (brute
    force over all m < 2^(n-w): rep = anchor + m p), ties to the smaller value (ring.hpp:77-90)."""
    lib = O.lib()
    for u in range(1 << f.w):
        rep = P.sparse_transform(u, f)
        assert lib.or_poly_mod(rep, f.modulus) == u
        cands = [lib.or_poly_mod(u, f.modulus) ^ lib.or_clmul(mm, f.modulus) for mm in range(1 << (f.n - f.w))]
        best = min(cands, key=lambda c: (bin(c).count("1"), c))
        assert bin(rep).count("1") == bin(best).count("1")
        assert rep == O.sparse_transform(u, ofield(f))


AOP_ESP = [P.FieldSpec(2, 3, 0, 1, 2, 0b111), P.FieldSpec.gf16_aop(), P.FieldSpec.gf64_esp(), P.FieldSpec.aop(10),
           P.FieldSpec.aop(12)]
KNOBS = ("PARTS", "PART_GROUP", "PART_CSE", "CSE_WINDOW", "PART_TEMPS")


@st.composite
def part_cases(draw):
    parity = draw(st.booleans())
    f = draw(st.sampled_from(AOP_ESP if parity else FIELDS))
    k = draw(st.integers(1, 7))
    r = draw(st.integers(1, 6))
    entries = draw(st.lists(st.integers(0, (1 << f.w) - 1), min_size=k * r, max_size=k * r))
    m = np.array(entries, dtype=np.uint16).reshape(r, k)
    knobs = {"PARTS": draw(st.integers(1, 4)), "PART_GROUP": draw(st.integers(1, 4)),
             "PART_CSE": draw(st.integers(0, 1)), "CSE_WINDOW": draw(st.sampled_from([0, 1, 2, 5])),
             "PART_TEMPS": draw(st.sampled_from([0, 3]))}
    group = draw(st.integers(0, 3))
    strip = draw(st.integers(1, 24))
    return f, int(parity), m, knobs, group, strip, draw(st.integers(0, 2**31))


@settings(max_examples=300, deadline=None)
@given(part_cases())
def test_output_parts_and_pair_sharing(case):
    """The programs the kernels actually run -- output parts (the staged kernel's warp groups, the
    split direct kernel's thread groups) with their fragment groups and windowed pair sharing --
    interpreted part by part, against the field oracle; both transforms."""
    import os
    f, kind, m, knobs, group, strip, seed = case
    rng = np.random.default_rng(seed)
    r, k = m.shape
    ins = [rng.integers(0, 256, f.w * strip, dtype=np.uint8) for _ in range(k)]
    want = O.apply_columns(ofield(f), m, ins, strip, kind=kind)
    saved = {n: os.environ.get("PYRIT_B200_" + n) for n in KNOBS + ("INTERPRET_PARTS",)}
    try:
        for n, v in knobs.items():
            os.environ["PYRIT_B200_" + n] = str(v)
        os.environ["PYRIT_B200_INTERPRET_PARTS"] = "1"
        plan = P.Plan.create(f, m, transform=P.TransformKind(kind), group=group)
        assert plan.stats()["parts"] == min(knobs["PARTS"], r)
        got = plan.interpret(ins, strip, outs=[np.full(f.w * strip, 0xA5, dtype=np.uint8) for _ in range(r)])
    finally:
        for n, v in saved.items():
            if v is None:
                os.environ.pop("PYRIT_B200_" + n, None)
            else:
                os.environ["PYRIT_B200_" + n] = v
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@settings(max_examples=200, deadline=None)
@given(part_cases())
def test_generic_kernel_bitmatrix(case):
    """The generic kernel's bitmatrix (Program::field_masks: the field code for the embedding, read off
    the program for the Parity transform) computes the same bytes as the oracle, evaluated on the
    host (PYRIT_B200_INTERPRET_GENERIC)."""
    import os
    f, kind, m, _knobs, group, strip, seed = case
    rng = np.random.default_rng(seed)
    r, k = m.shape
    ins = [rng.integers(0, 256, f.w * strip, dtype=np.uint8) for _ in range(k)]
    want = O.apply_columns(ofield(f), m, ins, strip, kind=kind)
    plan = P.Plan.create(f, m, transform=P.TransformKind(kind), group=group)
    os.environ["PYRIT_B200_INTERPRET_GENERIC"] = "1"
    try:
        got = plan.interpret(ins, strip, outs=[np.full(f.w * strip, 0x3C, dtype=np.uint8) for _ in range(r)])
    finally:
        os.environ.pop("PYRIT_B200_INTERPRET_GENERIC", None)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)

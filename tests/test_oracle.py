"""Pin the CPU oracle (oracle/pyrit_oracle.c) before trusting it.

(1) The reference's own known-answer tests, value for value (cited per test).
(2) Golden fixtures produced by the reference itself (tests/golden/make_golden.py).
(3) Live cross-checks against the reference compiled in place (oracle/_ref),
    when that library is present.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
ARR = np.load(os.path.join(HERE, "golden", "golden.npz"))
FIELDS = {1: O.GF256_R17, 4: O.GF16, 6: O.GF64, 8: O.GF256_R17, 10: O.GF1024, 12: O.GF4096}


def _has_ref():
    return os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libpyrit_ref.so"))


needs_ref = pytest.mark.skipif(not _has_ref(), reason="oracle/_ref not built (no reference tree)")


# ---------------------------------------------------------------- (1) KATs
def test_field_kats():
    # test_field.cpp: x^2 * x^3 = 1 and x * x^3 = 0xF in GF16 (AOP x^4+x^3+x^2+x+1)
    assert O.gf_mul(0x4, 0x8, O.GF16) == 1
    assert O.gf_mul(0x2, 0x8, O.GF16) == 0xF
    for f in (O.GF16, O.GF64, O.GF1024, O.GF4096, O.GF256_R17):
        for a in range(1, min(1 << f.w, 600)):
            assert O.gf_mul(a, O.gf_inv(a, f), f) == 1


def test_ring_kats():
    # test_ring.cpp:14-21: (1+x^2)(x+x^4) = x^3+x^4 in R_{2,5}; x^3 * x^7 = x in R_{2,9}
    assert O.ring_mul(0x05, 0x12, O.GF16) == 0x18
    assert O.ring_mul(0x008, 0x080, O.GF64) == 0x002
    # test_ring.cpp:88-98: sparse(x^2) = x^2, sparse(0) = 0, sparse(1) = 1; rep = u mod p, weight <= phi1's
    assert O.sparse_transform(0x4, O.GF16) == 0x4
    assert O.sparse_transform(0, O.GF16) == 0
    assert O.sparse_transform(1, O.GF16) == 1
    for f in (O.GF16, O.GF64, O.GF1024, O.GF4096, O.GF256_R17):
        for u in range(0, 1 << f.w, max(1, (1 << f.w) // 256)):
            rep = O.sparse_transform(u, f)
            assert O.lib().or_poly_mod(rep, f.modulus) == u
            assert rep < (1 << f.n)


def test_fold_table_matches_reference_rule_for_aop_esp():
    # transform.hpp:39-46: top coefficient w + j folds into every i with i % s == j
    for f in (O.GF16, O.GF64, O.GF1024, O.GF4096):
        fold = O.fold_table(f)
        for t in range(f.w, f.n):
            want = sum(1 << i for i in range(f.w) if i % f.s == t - f.w)
            assert fold[t - f.w] == want
    # phi_E_inv KATs (test_transforms.cpp:16-31): x^4 -> 0xF in GF16, x^6 -> 1 + x^3 in GF64
    assert O.fold_table(O.GF16)[0] == 0xF
    assert O.fold_table(O.GF64)[0] == 0x09
    # R_{2,17}: the general rule (x^t mod p), which the reference cannot express
    assert O.fold_table(O.GF256_R17)[0] == 0x139 & 0xFF


def test_hand_case_and_linearity():
    # test_codec.cpp:82-106: k=2, M=[1, x^2], d=(1, x^3) -> parity column 0 is 0
    m = np.array([[1, 0x4]], dtype=np.uint16)
    d0 = np.zeros(8, np.uint8)
    d1 = np.zeros(8, np.uint8)
    d0[0] |= 1  # column 0 of symbol 0 = 1 (strip 0 bit 0)
    d1[3 * 2] |= 1  # column 0 of symbol 1 = x^3 (strip 3 bit 0); strip = 2 bytes
    out = O.apply_columns(O.GF16, m, [d0, d1], 2)
    assert all(out[0][s * 2] & 1 == 0 for s in range(4))
    rng = np.random.default_rng(7)
    c = O.cauchy(3, 2, O.GF16)
    a = [rng.integers(0, 256, 16, dtype=np.uint8) for _ in range(3)]
    b = [rng.integers(0, 256, 16, dtype=np.uint8) for _ in range(3)]
    pa, pb = O.apply_columns(O.GF16, c, a, 4), O.apply_columns(O.GF16, c, b, 4)
    ps = O.apply_columns(O.GF16, c, [x ^ y for x, y in zip(a, b)], 4)
    for i in range(2):
        np.testing.assert_array_equal(ps[i], pa[i] ^ pb[i])


def test_cauchy_normalized_and_bounds():
    # test_matrix.cpp:23-44
    for f in (O.GF16, O.GF64):
        c = O.cauchy(6, 6, f)
        assert (c[0] == 1).all() and (c[:, 0] == 1).all()
    assert O.cauchy(1, 1, O.GF16)[0, 0] == 1
    with pytest.raises(O.OracleError) as e:
        O.cauchy(13, 4, O.GF16)
    assert e.value.rc == 3  # TooManySymbols


def test_invert_roundtrip_and_singular():
    rng = np.random.default_rng(37)
    for f in (O.GF16, O.GF64, O.GF4096):
        for _ in range(50):
            dim = int(rng.integers(1, 5))
            while True:
                m = rng.integers(0, 1 << f.w, (dim, dim)).astype(np.uint16)
                try:
                    mi = O.invert(m, f)
                    break
                except O.OracleError:
                    continue
            prod = np.zeros((dim, dim), dtype=np.uint32)
            for i in range(dim):
                for j in range(dim):
                    acc = 0
                    for t in range(dim):
                        acc ^= O.gf_mul(int(m[i, t]), int(mi[t, j]), f)
                    prod[i, j] = acc
            assert (prod == np.eye(dim, dtype=np.uint32)).all()
    with pytest.raises(O.OracleError) as e:
        O.invert(np.ones((2, 2), np.uint16), O.GF16)
    assert e.value.rc == 2  # Singular


def test_schedule_op_counts():
    # acceptance.cpp / SURVEY 8(a) a7: ring schedule region ops 52, 1430, 2808; widened R_{2,17} 816
    for f, k, r, want in ((O.GF16, 4, 2, 52), (O.GF1024, 12, 4, 1430), (O.GF4096, 16, 4, 2808),
                          (O.GF256_R17, 10, 4, 816)):
        c = O.cauchy(k, r, f)
        ss = f.w * 8
        data = [np.zeros(ss, np.uint8) for _ in range(k)]
        _, ops = O.ring_replay(f, c, data, 8, want_ops=True)
        assert ops == want


def test_fill_and_digest_twins():
    for seed, frag, begin, n, valid in ((0, 0, 0, 4096, 4096), (4, 15, 8 * 77, 1000 * 8, 8 * 77 + 3333),
                                        (3, 9, 0, 64, 10)):
        a = O.fill(seed, frag, n, valid=valid, begin=begin)
        b = O.fill_np(seed, frag, n, valid=valid, begin=begin)
        np.testing.assert_array_equal(a, b)
        assert O.digest(a, 5) == O.digest_np(a, 5)
    x = O.fill_np(1, 2, 8192)
    assert (O.digest_np(x[:4096], 0) + O.digest_np(x[4096:], 512)) % 2**64 == O.digest_np(x, 0)


# ------------------------------------------------------ (2) golden fixtures
@pytest.mark.parametrize("cfg", ["1", "2", "3", "4", "5"])
def test_golden_baseline_configs(cfg):
    g = GOLDEN["configs"][cfg]
    f = FIELDS[g["w"]] if g["w"] != 8 else O.GF256_R17
    c = O.cauchy(g["k"], g["r"], f)
    assert c.tolist() == g["cauchy"]
    if "reps" in g:
        assert [[O.sparse_transform(int(u), f) for u in row] for row in c] == g["reps"]
    strip = GOLDEN["strip_bytes"]
    data = [O.fill_np(g["seed"], j, f.w * strip) for j in range(g["k"])]
    want = ARR[f"cfg{cfg}_parity"]
    np.testing.assert_array_equal(np.stack(O.apply_columns(f, c, data, strip)), want)
    np.testing.assert_array_equal(np.stack(O.ring_replay(f, c, data, strip)), want)
    if "schedule_stats" in g:
        _, ops = O.ring_replay(f, c, data, strip, want_ops=True)
        assert ops == g["schedule_stats"]["total"]
    if "decode_matrix" in g:
        dm = O.decode_matrix(g["k"], g["r"], f, g["decode_survivors"])
        assert dm.tolist() == g["decode_matrix"]


def test_golden_small_codes_both_transforms():
    for key in GOLDEN["small"]:
        w = int(key.split("_")[1][1:])
        k = int(key.split("_")[2][1:])
        transform = int(key.split("_")[4][1:])
        f = O.GF16 if w == 4 else O.GF64
        data = ARR[key + "_data"]
        r = ARR[key + "_parity"].shape[0]
        c = O.cauchy(k, r, f)
        strip = data.shape[1] // f.w
        got = np.stack(O.apply_columns(f, c, list(data), strip, kind=transform))
        np.testing.assert_array_equal(got, ARR[key + "_parity"], err_msg=key)
        got2 = np.stack(O.ring_replay(f, c, list(data), strip, kind=transform))
        np.testing.assert_array_equal(got2, ARR[key + "_parity"], err_msg=key)


def test_golden_sparse_reps_all_elements():
    for w, reps in GOLDEN["sparse_reps"].items():
        f = FIELDS[int(w)]
        assert [O.sparse_transform(u, f) for u in range(1 << f.w)] == reps


def test_oracle_decode_roundtrip():
    f = O.GF256_R17
    k, r = 10, 4
    strip = 64
    data = [O.fill_np(3, j, f.w * strip) for j in range(k)]
    par = O.apply_columns(f, O.cauchy(k, r, f), data, strip)
    full = [x.copy() for x in data + par]
    work = [x.copy() for x in full]
    for e in (1, 6, 9, 10):
        work[e][:] = 0xAA
    O.decode(k, r, f, work, (1, 6, 9, 10), strip)
    for a, b in zip(work, full):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(O.OracleError) as e:
        O.decode(k, r, f, work, (0, 1, 2, 3, 4), strip)
    assert e.value.rc == 6  # InsufficientShards


# ------------------------------------------------ (3) live reference checks
@needs_ref
def test_live_reference_sparse_and_cauchy():
    for f in (O.GF16, O.GF64, O.GF1024, O.GF4096):
        for u in range(1 << f.w):
            assert O.sparse_transform(u, f) == O.ref_sparse_transform(u, f)
    for f, k, r in ((O.GF16, 4, 2), (O.GF256_R17, 10, 4), (O.GF1024, 12, 4), (O.GF4096, 16, 4), (O.GF64, 40, 20)):
        np.testing.assert_array_equal(O.cauchy(k, r, f), O.ref_cauchy(k, r, f))


@needs_ref
@pytest.mark.parametrize("f,k,r", [(O.GF16, 4, 2), (O.GF64, 6, 3), (O.GF1024, 12, 4), (O.GF4096, 16, 4),
                                   (O.GF256_R17, 10, 4)])
def test_live_reference_encode(f, k, r):
    rng = np.random.default_rng(k * 100 + r)
    ss = f.w * 64
    data = rng.integers(0, 256, (k, ss), dtype=np.uint8)
    c = O.cauchy(k, r, f)
    ring_ok = f.n <= 16
    want = O.ref_encode(f, k, r, np.ascontiguousarray(data.reshape(-1)), ss, crs=0 if ring_ok else 1).reshape(r, ss)
    np.testing.assert_array_equal(np.stack(O.apply_columns(f, c, list(data), ss // f.w)), want)
    np.testing.assert_array_equal(np.stack(O.ring_replay(f, c, list(data), ss // f.w)), want)
    if ring_ok:
        st = O.ref_schedule_stats(f, c)
        _, ops = O.ring_replay(f, c, list(data), ss // f.w, want_ops=True)
        assert ops == st["total"]
    else:
        # the reference's own ring encode is wrong on R_{2,17}
        bad = O.ref_encode(f, k, r, np.ascontiguousarray(data.reshape(-1)), ss).reshape(r, ss)
        assert not np.array_equal(bad, want)

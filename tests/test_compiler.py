"""Host side of the product on CPU: algebra through the C ABI and the ring
program compiler (executed by its host interpreter) against the oracle and the
reference's golden fixtures.  No device calls."""
from __future__ import annotations

import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from paper_1709_00178_b200.workloads import WORKLOADS
from tests.helpers import G16, G64, G256, G1024, G4096, ofield, oracle_encode, rand_symbols

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
ARR = np.load(os.path.join(HERE, "golden", "golden.npz"))


@pytest.mark.parametrize("f", [G16, G64, G1024, G4096])
def test_sparse_transform_equals_reference_for_every_element(f):
    reps = GOLDEN["sparse_reps"][str(f.w)]
    assert [P.sparse_transform(u, f) for u in range(1 << f.w)] == reps


def test_sparse_transform_widened_r17_self_consistent():
    f = G256
    of = ofield(f)
    for u in range(256):
        rep = P.sparse_transform(u, f)
        assert rep == O.sparse_transform(u, of)
        assert O.lib().or_poly_mod(rep, f.modulus) == u
        # minimal weight over the whole coset {u + m p : deg < 17}
        best = min(bin(u ^ O.lib().or_clmul(m, f.modulus)).count("1") for m in range(1 << 9))
        assert bin(rep).count("1") == best


def test_field_and_matrix_algebra():
    for f in (G16, G64, G256, G1024, G4096):
        of = ofield(f)
        for a in range(1, 1 << f.w, max(1, (1 << f.w) // 64)):
            assert P.gf_inv(a, f) == O.gf_inv(a, of)
            assert P.gf_mul(a, 3, f) == O.gf_mul(a, 3, of)
        assert P.fold_table(f) == O.fold_table(of)
    for cfg in ("1", "2", "3", "4", "5"):
        g = GOLDEN["configs"][cfg]
        wl = WORKLOADS[int(cfg)]
        assert P.cauchy_parity_matrix(wl.code).tolist() == g["cauchy"]
    g = GOLDEN["configs"]["4"]
    assert P.decode_matrix(WORKLOADS[4].code, g["decode_survivors"]).tolist() == g["decode_matrix"]


def test_errors_mirror_errc():
    with pytest.raises(P.PyritError) as e:
        P.cauchy_parity_matrix(P.CodeSpec(13, 4, G16))
    assert e.value.code == "TooManySymbols"
    with pytest.raises(P.PyritError) as e:
        P.cauchy_parity_matrix(P.CodeSpec(0, 4, G16))
    assert e.value.code == "InvalidArgument"
    with pytest.raises(P.PyritError) as e:
        P.Plan.create(G16, np.ones((2, 2), np.uint16) * 99)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(P.PyritError) as e:
        P.Plan.decode(P.CodeSpec(4, 2, G16), [0, 1, 2])
    assert e.value.code == "InsufficientShards"
    with pytest.raises(P.PyritError) as e:
        P.Plan.decode(P.CodeSpec(4, 2, G16), [9])
    assert e.value.code == "InvalidArgument"
    with pytest.raises(P.PyritError) as e:
        P.Plan.decode(P.CodeSpec(4, 2, G16), [1, 1])
    assert e.value.code == "InvalidArgument"
    with pytest.raises(P.PyritError):  # p does not divide x^n + 1
        P.gf_mul(1, 1, P.FieldSpec(4, 6, 0, 1, 4, 0x1F))


@pytest.mark.parametrize("cfg,ops,ones", [(1, 52, 44), (3, 1430, 1390), (5, 2808, 2760), (2, 816, 656)])
def test_reference_op_counts(cfg, ops, ones):
    """Region-op count of the equivalent compile_schedule (schedule.hpp:94-163) and matrix_ones."""
    st = P.Plan.encode(WORKLOADS[cfg].code).stats()
    assert st["ref_region_ops"] == ops
    assert st["matrix_ones"] == ones
    g = GOLDEN["configs"][str(cfg)]
    if "schedule_stats" in g:
        assert st["ref_region_ops"] == g["schedule_stats"]["total"]
        assert st["matrix_ones"] == g["schedule_stats"]["matrix_ones"]
    assert st["xors"] < st["naive_xors"]  # pair sharing never adds work


def test_dense_representatives_never_cheaper():
    # test_schedule.cpp:159-173
    for f in (G16, G64):
        for k in range(1, 7):
            for r in range(1, 7):
                c = P.cauchy_parity_matrix(P.CodeSpec(k, r, f))
                sp = P.Plan.create(f, c, rep=P.RingRep.Sparse).stats()
                de = P.Plan.create(f, c, rep=P.RingRep.Dense).stats()
                assert sp["ref_region_ops"] <= de["ref_region_ops"]
                assert sp["matrix_ones"] <= de["matrix_ones"]


@pytest.mark.parametrize("cfg", ["1", "2", "3", "5"])
def test_compiled_program_matches_golden(cfg):
    g = GOLDEN["configs"][cfg]
    wl = WORKLOADS[int(cfg)]
    strip = GOLDEN["strip_bytes"]
    data = [O.fill_np(g["seed"], j, wl.fld.w * strip) for j in range(wl.k)]
    for group in (1, 2, 0):
        for cse in (True,):
            plan = P.Plan.create(wl.fld, P.cauchy_parity_matrix(wl.code), group=group)
            got = np.stack(plan.interpret(data, strip))
            np.testing.assert_array_equal(got, ARR[f"cfg{cfg}_parity"])


def test_compiled_windows():
    """Windows [off, off+len) of every strip equal the same window of a full apply."""
    wl = WORKLOADS[5]
    strip = 256
    data = [O.fill_np(4, j, wl.fld.w * strip) for j in range(wl.k)]
    plan = P.Plan.encode(wl.code)
    full = plan.interpret(data, strip)
    part = [np.zeros_like(x) for x in full]
    for lo, hi in ((0, 48), (48, 200), (200, 256)):
        plan.interpret(data, strip, lo, hi - lo, outs=part)
    for a, b in zip(full, part):
        np.testing.assert_array_equal(a, b)


def test_small_codes_both_transforms_golden():
    for key in GOLDEN["small"]:
        w = int(key.split("_")[1][1:])
        k = int(key.split("_")[2][1:])
        transform = int(key.split("_")[4][1:])
        f = G16 if w == 4 else G64
        data = ARR[key + "_data"]
        want = ARR[key + "_parity"]
        code = P.CodeSpec(k, want.shape[0], f, P.TransformKind(transform))
        plan = P.Plan.create(f, P.cauchy_parity_matrix(code), transform=transform)
        got = np.stack(plan.interpret(list(data), data.shape[1] // f.w))
        np.testing.assert_array_equal(got, want, err_msg=key)


@pytest.mark.parametrize("grid", [(4, 2, G16), (6, 3, G16), (6, 3, G64)])
@pytest.mark.parametrize("kind", [0, 1])
def test_every_erasure_pattern_repairs(grid, kind):
    """test_codec.cpp:108-143, every pattern of weight <= r, through the fused repair program."""
    k, r, f = grid
    code = P.CodeSpec(k, r, f, P.TransformKind(kind))
    ss = int(np.lcm(f.w, 8)) * 2
    strip = ss // f.w
    data = rand_symbols(k, ss, 911)
    full = np.concatenate([data, oracle_encode(f, P.cauchy_parity_matrix(code), data, kind=kind)])
    for wgt in range(1, r + 1):
        for erased in itertools.combinations(range(k + r), wgt):
            plan = P.Plan.decode(code, erased)
            outs = plan.interpret([full[s] for s in plan.survivors], strip)
            assert plan.outputs == sorted(e for e in erased if e < k) + sorted(e for e in erased if e >= k)
            for o, arr in zip(plan.outputs, outs):
                np.testing.assert_array_equal(arr, full[o], err_msg=f"{erased}")


def test_production_size_codes_random_patterns():
    """test_codec.cpp:145-180: (8,4) GF16, (40,20) GF64 embedding, (20,40) GF64 parity."""
    rng = np.random.default_rng(913)
    for k, r, f, kind in ((8, 4, G16, 0), (40, 20, G64, 0), (20, 40, G64, 1)):
        code = P.CodeSpec(k, r, f, P.TransformKind(kind))
        ss = int(np.lcm(f.w, 8))
        strip = ss // f.w
        data = rand_symbols(k, ss, k + r)
        full = np.concatenate([data, oracle_encode(f, P.cauchy_parity_matrix(code), data, kind=kind)])
        for _ in range(6):
            erased = rng.permutation(k + r)[: 1 + rng.integers(r)].tolist()
            plan = P.Plan.decode(code, erased)
            outs = plan.interpret([full[s] for s in plan.survivors], strip)
            for o, arr in zip(plan.outputs, outs):
                np.testing.assert_array_equal(arr, full[o])


def test_config4_fused_repair_matches_two_pass_reference_semantics():
    """Fused rows (erased data of A^-1, then C_i A^-1) == decode()'s two passes (codec.hpp:269-283)."""
    wl = WORKLOADS[4]
    f = wl.fld
    strip = 64
    data = np.stack([O.fill_np(3, j, f.w * strip) for j in range(wl.k)])
    full = np.concatenate([data, oracle_encode(f, P.cauchy_parity_matrix(wl.code), data)])
    surv, outs, m = P.repair_matrix(wl.code, wl.erased)
    assert surv.tolist() == [0, 2, 3, 4, 5, 7, 8, 11, 12, 13]
    assert outs.tolist() == [1, 6, 9, 10]
    plan = P.Plan.decode(wl.code, wl.erased)
    got = plan.interpret([full[s] for s in plan.survivors], strip)
    for o, arr in zip(plan.outputs, got):
        np.testing.assert_array_equal(arr, full[o])
    # oracle two-pass decode agrees
    work = [x.copy() for x in full]
    for e in wl.erased:
        work[e][:] = 0
    O.decode(wl.k, wl.m, ofield(f), work, wl.erased, strip)
    np.testing.assert_array_equal(np.stack(work), full)


def test_generated_source_is_straight_line():
    name, src = P.Plan.encode(WORKLOADS[5].code).source(1)
    assert name.startswith("pyrit_ring_k16_e4_w12_n13")
    assert "__launch_bounds__" in src and "ld.global.nc" in src and "st.global.cs" in src
    assert "while (b < a.nb)" in src and src.count("LD(") == 16 * 12 + 1  # one per strip (+ macro)


@pytest.mark.parametrize("f,k,r", [(G16, 4, 2), (G64, 6, 3), (G256, 10, 4), (G1024, 12, 4), (G4096, 16, 4)])
def test_crs_bitmatrix_program(f, k, r):
    """rep=2: the Cauchy-RS bitmatrix program (compile_crs_schedule, schedule.hpp:168-203)
    computes the plain field code, and its op count equals the reference's CRS schedule."""
    c = P.CodeSpec(k, r, f)
    m = P.cauchy_parity_matrix(c)
    plan = P.Plan.create(f, m, rep=P.RingRep.Crs)
    ss = f.w * 40
    data = rand_symbols(k, ss, k + r)
    got = np.stack(plan.interpret(list(data), ss // f.w))
    np.testing.assert_array_equal(got, oracle_encode(f, m, data))
    st = plan.stats()
    want = O.ref_schedule_stats(ofield(f), m, crs=1) if f.n <= 16 else None
    if want:  # the reference's CRS compiler works for every field with 16-bit ring elements
        assert st["ref_region_ops"] == want["total"] and st["matrix_ones"] == want["matrix_ones"]
    assert plan.key() != P.Plan.create(f, m).key() and "crs" in plan.key()
    with pytest.raises(P.PyritError):
        P.Plan.create(f, m, P.TransformKind.Parity, rep=P.RingRep.Crs)

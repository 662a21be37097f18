"""Shard container + file codec (container.hpp), mirroring the reference's
proj/tests/test_container.cpp case by case.

CPU tests pin the header/CRC code of libpyrit_b200.so (pure host code, no
device) and the oracle's restated file codec against the reference compiled
in place (oracle/_ref).  GPU tests (-m gpu) run the product's encode_file /
decode_file -- stripe batches through the sm_100a kernel -- and compare the
shard files byte for byte with the reference (gf16/gf64 sets, the only ones
the reference's field ids can record) and with the oracle (BASELINE fields).
"""
from __future__ import annotations

import filecmp
import itertools
import os
import random

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from tests.helpers import G16, G64, G256, G1024, G4096, ofield

ERR = {name: i + 1 for i, name in enumerate(P._lib.ERRC)}


def random_bytes(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 256, n, dtype=np.uint8)


def spit(path, data: np.ndarray) -> None:
    data.tofile(str(path))


def slurp(path) -> bytes:
    with open(str(path), "rb") as f:
        return f.read()


def code(k, r, f, kind=0):
    return P.CodeSpec(k, r, f, P.TransformKind(kind))


# ------------------------------------------------------------------ CPU pins
def test_crc32_check_value():
    """test_container.cpp:46-51: CRC-32 of "123456789" is 0xCBF43926; empty -> 0."""
    assert P.crc32(b"123456789") == 0xCBF43926
    assert P.crc32(b"") == 0
    assert O.crc32(b"123456789") == 0xCBF43926
    for n in (1, 7, 25, 300):
        b = random_bytes(n, n).tobytes()
        assert P.crc32(b) == O.crc32(b) == O.ref().ref_crc32(b, n)


def test_header_round_trip_matches_reference():
    """test_container.cpp:53-72, plus byte equality with the reference serializer."""
    h = P.ShardHeader(1, 1, 1, 20, 40, 59, 24, 123456789)
    b = P.serialize_header(h)
    assert len(b) == P.HEADER_SIZE == 29 and b[:4] == b"PYRT"
    assert P.parse_header(b) == h
    assert h.stripe_count() == (123456789 + 20 * 24 - 1) // (20 * 24)
    assert b == O.ref_serialize_header(1, 1, 20, 40, 59, 24, 123456789) == O.serialize_header(1, 1, 20, 40, 59, 24,
                                                                                              123456789)
    rng = random.Random(7)
    for _ in range(200):
        args = (rng.randrange(2), rng.randrange(2), rng.randrange(1, 30), rng.randrange(30), rng.randrange(60),
                8 * rng.randrange(1, 1000), rng.randrange(1 << 40))
        ours = P.serialize_header(P.ShardHeader(1, *args))
        assert ours == O.ref_serialize_header(*args)


def test_parse_rejects_corruption_with_typed_errors():
    """test_container.cpp:74-120."""
    good = P.serialize_header(P.ShardHeader(1, 0, 0, 4, 2, 0, 16, 64))

    def mutate(at, v):
        b = bytearray(good)
        b[at] = v
        return bytes(b)

    cases = [(mutate(0, ord("X")), "BadHeader"), (mutate(4, 9), "BadHeader"), (mutate(13, 0x11), "ChecksumError"),
             (good[:5], "BadHeader")]
    junk = bytearray(good)
    junk[5] = 77  # no such field id, checksum fixed up
    junk[25:29] = O.crc32(bytes(junk[:25])).to_bytes(4, "little")
    cases.append((bytes(junk), "BadHeader"))
    for b, want in cases:
        with pytest.raises(P.PyritError) as ei:
            P.parse_header(b)
        assert ei.value.code == want
        with pytest.raises(O.OracleError) as ej:
            O.ref_parse_header(b)
        assert ej.value.rc == ERR[want]


def test_header_fuzzing_matches_reference():
    """test_container.cpp:122-135: never crashes; here also the same verdict as the
    reference for every input (field ids 2..4 are this library's extension)."""
    rng = random.Random(4242)
    for rnd in range(2000):
        b = bytearray(rng.randrange(256) for _ in range(rng.randrange(40)))
        if rnd % 3 == 0 and len(b) >= 4:
            b[:4] = b"PYRT"
        if rnd % 5 == 0 and len(b) >= 29:  # valid checksum so the semantic checks run
            b[4] = 1
            b[25:29] = O.crc32(bytes(b[:25])).to_bytes(4, "little")
        b = bytes(b)
        try:
            ours = P.parse_header(b)
            ours_rc = 0
        except P.PyritError as e:
            ours, ours_rc = None, e.rc
        try:
            theirs = O.ref_parse_header(b)
            ref_rc = 0
        except O.OracleError as e:
            theirs, ref_rc = None, e.rc
        if ours is not None and ours.field >= 2:
            assert ref_rc == ERR["BadHeader"]  # unknown to the reference
            continue
        assert ours_rc == ref_rc, b.hex()
        if ours is not None:
            assert tuple(getattr(ours, k) for k in ("version", "field", "transform", "k", "r", "shard_index",
                                                    "symbol_size", "original_length")) == theirs


def test_field_ids():
    assert [P.field_id(f) for f in (G16, G64, G256, G1024, G4096)] == [0, 1, 2, 3, 4]
    assert P.field_from_id(0) == G16 and P.field_from_id(1) == P.FieldSpec(6, 9, 1, 3, 2, 0x49)
    with pytest.raises(P.PyritError) as ei:
        P.field_from_id(5)
    assert ei.value.code == "BadHeader"
    with pytest.raises(P.PyritError) as ei:
        P.field_id(P.FieldSpec(4, 5, 0, 1, 4, 0x13 | 0))  # not a supported field
    assert ei.value.rc in (ERR["InvalidArgument"],)


def test_shard_path():
    assert P.shard_path("/x/y/input.bin", "/out", 7) == "/out/input.bin.s007.pyrit"
    assert os.path.basename(P.shard_path("a.b", "d", 123)) == O.shard_name("a.b", 123) == "a.b.s123.pyrit"


ORACLE_CASES = [  # (k, r, field, kind, symbol_size, length, seed) -- test_container.cpp cases
    (4, 2, O.GF16, 0, 128, 10000, 99),
    (3, 6, O.GF64, 1, 48, 4321, 100),
    (2, 1, O.GF16, 0, 64, 500, 1),
    (4, 2, O.GF16, 0, 64, 3000, 3),
    (2, 2, O.GF16, 0, 32, 0, 0),
] + [(3, 2, O.GF16, 0, 16, n, n) for n in (1, 63, 64, 65, 4095)]


@pytest.mark.parametrize("case", ORACLE_CASES)
def test_oracle_file_codec_matches_reference(tmp_path, case):
    """The oracle's restated encode_file/decode_file == the reference's, byte for byte."""
    k, r, f, kind, ss, n, seed = case
    payload = random_bytes(n, seed)
    spit(tmp_path / "input.bin", payload)
    O.ref_encode_file(tmp_path / "input.bin", tmp_path / "ref", k, r, f, ss, kind)
    ours = O.encode_file(tmp_path / "input.bin", tmp_path / "ora", k, r, f, ss, kind)
    for p in ours:
        assert filecmp.cmp(p, str(tmp_path / "ref" / os.path.basename(p)), shallow=False)
    surv = ours[r:]  # drop the first r shards (all data when r <= k)
    O.ref_decode_file(surv, tmp_path / "out_ref.bin")
    O.decode_file(surv, tmp_path / "out_ora.bin", k, r, f, ss, n, kind)
    assert slurp(tmp_path / "out_ref.bin") == slurp(tmp_path / "out_ora.bin") == payload.tobytes()


# ------------------------------------------------------------ GPU file codec
REF_FILE_CASES = [  # gf16/gf64: the reference itself is the oracle (byte-identical shard files)
    (4, 2, G16, 0, 128, 10000, 99),
    (3, 6, G64, 1, 48, 4321, 100),
    (2, 1, G16, 0, 64, 500, 1),
    (2, 1, G16, 1, 64, 500, 2),
    (4, 2, G16, 0, 64, 3000, 3),
    (2, 2, G16, 0, 32, 0, 0),
    (8, 4, G16, 0, 4096, 1 << 20, 5),
    (10, 5, G64, 0, 4104, 777777, 6),
] + [(3, 2, G16, 0, 16, n, n) for n in (1, 63, 64, 65, 4095)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", REF_FILE_CASES)
def test_encode_file_byte_identical_to_reference(cuda, tmp_path, case):
    k, r, f, kind, ss, n, seed = case
    payload = random_bytes(n, seed)
    spit(tmp_path / "input.bin", payload)
    ours = P.encode_file(tmp_path / "input.bin", tmp_path / "gpu", code(k, r, f, kind), ss)
    O.ref_encode_file(tmp_path / "input.bin", tmp_path / "ref", k, r, ofield(f), ss, kind)
    assert len(ours) == k + r
    for p in ours:
        assert os.path.getsize(p) == 29 + (0 if n == 0 else -(-n // (k * ss))) * ss
        assert filecmp.cmp(p, str(tmp_path / "ref" / os.path.basename(p)), shallow=False), p
    # and the reference decodes the GPU's shards
    O.ref_decode_file(ours[r:], tmp_path / "ref_out.bin")
    assert slurp(tmp_path / "ref_out.bin") == payload.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("f,k,r", [(G256, 10, 4), (G1024, 12, 4), (G4096, 16, 4), (G4096, 5, 3)])
def test_encode_file_baseline_fields_vs_oracle(cuda, tmp_path, f, k, r):
    """Fields the reference cannot record in a header (or encode, R_{2,17}): pinned to the oracle."""
    ss = f.w * 8 * 37  # odd strip (37*8 bytes): exercises the non-staged kernels
    n = 3 * k * ss + 1234
    payload = random_bytes(n, k)
    spit(tmp_path / "in.bin", payload)
    ours = P.encode_file(tmp_path / "in.bin", tmp_path / "gpu", code(k, r, f), ss)
    want = O.encode_file(tmp_path / "in.bin", tmp_path / "ora", k, r, ofield(f), ss)
    for a, b in zip(ours, want):
        assert filecmp.cmp(a, b, shallow=False), a
    rng = random.Random(k)
    for _ in range(3):
        erased = set(rng.sample(range(k + r), r))
        P.decode_file([p for i, p in enumerate(ours) if i not in erased], tmp_path / "out.bin")
        assert slurp(tmp_path / "out.bin") == payload.tobytes()


@pytest.mark.gpu
def test_decode_file_every_erasure_pattern(cuda, tmp_path):
    """test_container.cpp:137-177 generalised: every survivor set of size >= k."""
    payload = random_bytes(10000, 99)
    spit(tmp_path / "input.bin", payload)
    c = code(4, 2, G16)
    shards = P.encode_file(tmp_path / "input.bin", tmp_path, c, 128)
    for keep in range(4, 7):
        for surv in itertools.combinations(range(6), keep):
            out = tmp_path / "out.bin"
            P.decode_file([shards[i] for i in surv], out)
            assert slurp(out) == payload.tobytes(), surv
    # k-1 shards is not enough
    with pytest.raises(P.PyritError) as ei:
        P.decode_file([shards[0], shards[2], shards[4]], tmp_path / "out.bin")
    assert ei.value.code == "InsufficientShards"
    # duplicate shard paths do not double-count
    with pytest.raises(P.PyritError) as ei:
        P.decode_file([shards[0], shards[0], shards[1], shards[2]], tmp_path / "out.bin")
    assert ei.value.code == "InsufficientShards"
    # re-encoding is byte-identical
    again = P.encode_file(tmp_path / "input.bin", tmp_path / "again", c, 128)
    for a, b in zip(shards, again):
        assert slurp(a) == slurp(b)


@pytest.mark.gpu
def test_decode_file_errors_match_reference(cuda, tmp_path):
    """test_container.cpp:190-234: mixed sets, corrupt headers, truncation, missing files."""
    spit(tmp_path / "a.bin", random_bytes(500, 1))
    spit(tmp_path / "b.bin", random_bytes(500, 2))
    sa = P.encode_file(tmp_path / "a.bin", tmp_path, code(2, 1, G16), 64)
    sb = P.encode_file(tmp_path / "b.bin", tmp_path / "other", code(2, 1, G16, 1), 64)
    cases = [([sa[0], sb[1]], "HeaderMismatch")]
    spit(tmp_path / "c.bin", random_bytes(3000, 3))
    sc = P.encode_file(tmp_path / "c.bin", tmp_path / "c", code(4, 2, G16), 64)
    flipped = tmp_path / "flipped.pyrit"
    b = bytearray(slurp(sc[1]))
    b[7] ^= 0xFF
    flipped.write_bytes(bytes(b))
    cases.append(([sc[0], str(flipped), *sc[2:]], "ChecksumError"))
    trunc = tmp_path / "trunc.pyrit"
    trunc.write_bytes(slurp(sc[1])[:-1])
    cases.append(([sc[0], str(trunc), *sc[2:]], "BadHeader"))
    cases.append(([str(tmp_path / "nope.pyrit"), *sc[1:]], "IoError"))
    cases.append(([], "InsufficientShards"))
    for paths, want in cases:
        with pytest.raises(P.PyritError) as ei:
            P.decode_file(paths, tmp_path / "out.bin")
        assert ei.value.code == want, (paths, want)
        if paths:
            with pytest.raises(O.OracleError) as ej:
                O.ref_decode_file(paths, tmp_path / "out_ref.bin")
            assert ej.value.rc == ERR[want]


@pytest.mark.gpu
def test_empty_file(cuda, tmp_path):
    """test_container.cpp:238-247."""
    spit(tmp_path / "empty.bin", np.zeros(0, np.uint8))
    shards = P.encode_file(tmp_path / "empty.bin", tmp_path, code(2, 2, G16), 32)
    assert len(shards) == 4 and all(os.path.getsize(p) == 29 for p in shards)
    P.decode_file([shards[0], shards[3]], tmp_path / "out.bin")
    assert slurp(tmp_path / "out.bin") == b""


@pytest.mark.gpu
def test_file_pipeline_many_chunks(cuda, tmp_path):
    """Small pipeline chunks: many batches rotate through the three stages."""
    from paper_1709_00178_b200 import _lib as L
    lib = L.load()
    payload = random_bytes(5 * 1000 * 4096 + 77, 11)
    spit(tmp_path / "big.bin", payload)
    c = code(5, 3, G16)
    L.check(lib.pyrit_set_file_chunk(3 * 5 * 4096))  # 3 stripes per launch
    try:
        ours = P.encode_file(tmp_path / "big.bin", tmp_path / "gpu", c, 4096)
        P.decode_file([ours[i] for i in (1, 3, 5, 6, 7)], tmp_path / "out.bin")
    finally:
        L.check(lib.pyrit_set_file_chunk(0))
    assert slurp(tmp_path / "out.bin") == payload.tobytes()
    O.ref_encode_file(tmp_path / "big.bin", tmp_path / "ref", 5, 3, O.GF16, 4096)
    for p in ours:
        assert filecmp.cmp(p, str(tmp_path / "ref" / os.path.basename(p)), shallow=False)


# ------------------------------------------------------ stripe-batch kernels
@pytest.mark.gpu
@pytest.mark.parametrize("f,k,r,ss,nb", [
    (G16, 4, 2, 4096, 37),      # strip 1024: staged kernel
    (G16, 4, 2, 128, 1000),     # strip 32: direct kernel, 8 words per stripe
    (G64, 6, 3, 4104, 19),      # strip 684 (4-byte words)
    (G4096, 16, 4, 4104, 23),   # strip 342: byte mode
    (G256, 10, 4, 8 * 1024, 9),  # R_{2,17}, strip 1 KiB
    (G1024, 12, 4, 10 * 160, 31),
])
def test_encode_decode_batch_vs_oracle(cuda, f, k, r, ss, nb):
    import torch
    c = code(k, r, f)
    data = random_bytes(nb * k * ss, ss + nb).reshape(nb, k * ss)
    d = torch.from_numpy(data).to(cuda)
    par = P.encode_batch(d, c, ss)
    torch.cuda.synchronize()
    got = par.cpu().numpy()
    m = P.cauchy_parity_matrix(c)
    of = ofield(f)
    for b in range(nb):
        want = O.ring_replay(of, m, [data[b, j * ss:(j + 1) * ss].copy() for j in range(k)], ss // f.w)
        for i in range(r):
            np.testing.assert_array_equal(got[i, b], want[i], err_msg=f"stripe {b} parity {i}")
    # repair in place across the batch
    full = torch.cat([d.view(nb, k, ss).transpose(0, 1), par], 0).contiguous()  # (k + r, nb, ss)
    ref = full.clone()
    erased = sorted(random.Random(nb).sample(range(k + r), r))
    full[erased] = 0
    P.decode_batch(full, erased, c)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)


# ------------------------------------------- file codec validation (no device)
def test_file_codec_validation_before_any_device_work(tmp_path):
    """encode_file / decode_file reject bad arguments and damaged shard sets with the
    reference's error codes before touching a GPU (container.hpp:170-172, :229-275)."""
    spit(tmp_path / "in.bin", random_bytes(1000, 1))
    with pytest.raises(P.PyritError) as ei:
        P.encode_file(tmp_path / "in.bin", tmp_path / "o", code(4, 2, G16), 12)  # not a multiple of 8
    assert ei.value.code == "BufferShape"
    with pytest.raises(P.PyritError) as ei:
        P.encode_file(tmp_path / "in.bin", tmp_path / "o", code(4, 20, G16), 16)  # k + r > 16
    assert ei.value.code == "TooManySymbols"
    with pytest.raises(P.PyritError) as ei:
        P.encode_file(tmp_path / "missing.bin", tmp_path / "o", code(4, 2, G16), 16)
    assert ei.value.code == "IoError"
    with pytest.raises(P.PyritError) as ei:
        P.decode_file([], tmp_path / "out.bin")
    assert ei.value.code == "InsufficientShards"
    with pytest.raises(P.PyritError) as ei:
        P.decode_file([tmp_path / "nope.pyrit"], tmp_path / "out.bin")
    assert ei.value.code == "IoError"
    # shard files written by the reference (no GPU involved) feed the validation paths
    shards = O.encode_file(tmp_path / "in.bin", tmp_path / "ref", 4, 2, O.GF16, 64)
    bad = tmp_path / "bad.pyrit"
    b = bytearray(slurp(shards[0]))
    b[0] = ord("X")
    bad.write_bytes(bytes(b))
    with pytest.raises(P.PyritError) as ei:
        P.decode_file([str(bad)], tmp_path / "out.bin")
    assert ei.value.code == "BadHeader"
    with pytest.raises(P.PyritError) as ei:
        P.decode_file(shards[:3], tmp_path / "out.bin")  # k - 1 distinct shards
    assert ei.value.code == "InsufficientShards"

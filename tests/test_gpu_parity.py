"""GPU parity: the fused sm_100a kernels vs the CPU oracle, bit for bit.

Every call goes through libpyrit_b200.so (C ABI): device buffers are torch CUDA
tensors, results are copied back and compared with oracle/ (the plain-C
restatement, itself pinned against the reference in test_oracle.py).
"""
from __future__ import annotations

import itertools
import random

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from paper_1709_00178_b200 import _lib as L
from paper_1709_00178_b200.workloads import WORKLOADS, shard
from tests.helpers import G16, G64, G256, G1024, G4096, ofield, oracle_encode, oracle_ring, rand_symbols, seeded_symbols

pytestmark = pytest.mark.gpu


def dev_encode(cuda, code, data: np.ndarray) -> np.ndarray:
    import torch
    d = torch.from_numpy(data).to(cuda)
    out = P.encode(d, code)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def dev_decode(cuda, code, symbols: np.ndarray, erased) -> np.ndarray:
    import torch
    d = torch.from_numpy(symbols).to(cuda)
    P.decode(d, erased, code)
    torch.cuda.synchronize()
    return d.cpu().numpy()


def test_library_is_the_native_one(cuda):
    lib = L.load()
    assert b"sm_100a" in lib.pyrit_version()


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_baseline_encode_small(cuda, cfg):
    """BASELINE configs at a reduced fragment size: GPU == ring oracle == field oracle."""
    wl = WORKLOADS[cfg]
    f = wl.fld
    ss = f.w * 4096
    data = seeded_symbols(wl.k, ss, f.w, wl.seed)
    C = P.cauchy_parity_matrix(wl.code)
    got = dev_encode(cuda, wl.code, data)
    want = oracle_ring(f, C, data)
    np.testing.assert_array_equal(got, want)
    # field oracle (codec.hpp:444) on a window of every strip
    strip = ss // f.w
    outs = O.apply_columns(O.Field(f.w, f.n, f.kind, f.s, f.r_esp, f.modulus), C, list(data), strip, off=512,
                           length=256)
    for i in range(wl.m):
        for s in range(f.w):
            np.testing.assert_array_equal(got[i][s * strip + 512: s * strip + 768],
                                          outs[i][s * strip + 512: s * strip + 768])


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_encode_full_size(cuda, cfg):
    """Configs 1 and 2 at their full BASELINE size, every byte against the ring oracle."""
    wl = WORKLOADS[cfg]
    data = seeded_symbols(wl.k, wl.frag, wl.fld.w, wl.seed, valid=wl.valid)
    got = dev_encode(cuda, wl.code, data)
    want = oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("erased", [(1, 6, 9, 10), (0, 1, 2, 3), (10, 11, 12, 13), (2,), (0, 13)])
def test_config4_decode(cuda, erased):
    """Config 4 geometry (GF(2^8) in R_{2,17}, k=10, m=4): repair bit-exact, parity included."""
    wl = WORKLOADS[4]
    ss = wl.fld.w * 8192
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    parity = oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data)
    full = np.concatenate([data, parity])
    work = full.copy()
    work[list(erased)] = 0xAA
    got = dev_decode(cuda, wl.code, work, erased)
    np.testing.assert_array_equal(got, full)
    # and the C oracle's decode (codec.hpp:241 restated) agrees on a window
    work2 = full.copy()
    work2[list(erased)] = 0x55
    syms = [work2[i] for i in range(len(work2))]
    strip = ss // wl.fld.w
    O.decode(wl.k, wl.m, O.Field(8, 17, 0, 1, 8, 0x139), syms, erased, strip, off=0, length=strip)
    np.testing.assert_array_equal(np.stack(syms), full)


@pytest.mark.parametrize("spec", [G16, G64])
@pytest.mark.parametrize("kind", [0, 1])
def test_all_small_codes_match_oracle(cuda, spec, kind):
    """test_codec.cpp:53-80 / test_schedule.cpp:104-136 grid: k, r in [1,5], both transforms."""
    rng = random.Random(101 + kind)
    for k in range(1, 6):
        for r in range(1, 6):
            code = P.CodeSpec(k, r, spec, P.TransformKind(kind))
            ss = int(np.lcm(spec.w, 8)) * (1 + rng.randrange(3)) * 8
            data = rand_symbols(k, ss, rng.randrange(1 << 30))
            C = P.cauchy_parity_matrix(code)
            got = dev_encode(cuda, code, data)
            want = oracle_encode(spec, C, data, kind=kind)
            np.testing.assert_array_equal(got, want, err_msg=f"k={k} r={r} kind={kind}")


@pytest.mark.parametrize("grid", [(4, 2, G16), (6, 3, G16), (6, 3, G64)])
@pytest.mark.parametrize("kind", [0, 1])
def test_decode_erasure_patterns(cuda, grid, kind):
    """test_codec.cpp:108-143: erasure patterns of weight <= r repair bit-exact (sampled on GPU;
    every pattern is covered through the program interpreter in test_compiler.py)."""
    k, r, spec = grid
    code = P.CodeSpec(k, r, spec, P.TransformKind(kind))
    ss = int(np.lcm(spec.w, 8)) * 16
    data = rand_symbols(k, ss, 911)
    full = np.concatenate([data, oracle_encode(spec, P.cauchy_parity_matrix(code), data, kind=kind)])
    pats = [c for wgt in range(1, r + 1) for c in itertools.combinations(range(k + r), wgt)]
    rng = random.Random(7)
    for erased in rng.sample(pats, min(len(pats), 24)):
        work = full.copy()
        work[list(erased)] = 0xAA
        np.testing.assert_array_equal(dev_decode(cuda, code, work, erased), full, err_msg=str(erased))


def test_odd_strip_sizes_byte_mode(cuda):
    """Strips that are not word multiples (SymbolBuffer allows any multiple of lcm(w, 8))."""
    for spec, k, r in [(G16, 4, 2), (G64, 5, 3), (G256, 10, 4), (G4096, 16, 4)]:
        code = P.CodeSpec(k, r, spec)
        for mult in (3, 171):  # strips of 6/12/3/6 bytes and 342/684/171/342 (u8 / u16 elements)
            ss = int(np.lcm(spec.w, 8)) * mult
            data = rand_symbols(k, ss, 5)
            np.testing.assert_array_equal(dev_encode(cuda, code, data),
                                          oracle_encode(spec, P.cauchy_parity_matrix(code), data))
    # the 2-byte element kernel is the one a 342-byte strip takes
    code = P.CodeSpec(16, 4, G4096)
    dev_encode(cuda, code, rand_symbols(16, 4104, 6))
    assert "_H0" in P.Plan.last_launch()["kernel"]


def test_u16_kernel_windows_and_batches(cuda):
    """The u16-element direct kernel on 2-byte aligned strips, windows and stripe pitches (odd and even
    u16 counts), against the oracle; nothing outside the outputs is written."""
    import torch
    rng = np.random.default_rng(77)
    for spec, k, r in [(G4096, 16, 4), (G1024, 12, 4), (G256, 10, 4)]:
        code = P.CodeSpec(k, r, spec)
        m = P.cauchy_parity_matrix(code)
        plan = P.Plan.encode(code)
        for strip, off, length, nb in [(342, 0, 342, 1), (342, 2, 338, 3), (1026, 6, 1018, 2), (2050, 0, 2050, 4)]:
            sym = spec.w * strip
            pitch_in, pitch_out = k * sym + 2, r * sym + 6  # 2-byte aligned stripe pitches
            buf_in = rng.integers(0, 256, nb * pitch_in + 16, dtype=np.uint8)
            d = torch.from_numpy(buf_in).to(cuda)
            o = torch.full((nb * pitch_out + 16,), 0x77, dtype=torch.uint8, device=cuda)
            base_in, base_out = d.data_ptr() + 2, o.data_ptr() + 2
            plan.apply_batch([base_in + j * sym for j in range(k)], [base_out + i * sym for i in range(r)], strip, nb,
                             pitch_in, pitch_out, off, length, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert "_H0" in P.Plan.last_launch()["kernel"], P.Plan.last_launch()
            got = o.cpu().numpy()
            for b in range(nb):
                ins = [buf_in[2 + b * pitch_in + j * sym: 2 + b * pitch_in + (j + 1) * sym].copy() for j in range(k)]
                want = O.ring_replay(ofield(spec), m, ins, strip, off=off, length=length,
                                     outs=[np.full(sym, 0x77, dtype=np.uint8) for _ in range(r)])
                for i in range(r):
                    at = 2 + b * pitch_out + i * sym
                    np.testing.assert_array_equal(got[at: at + sym], want[i], err_msg=f"{spec.w} {strip} {b} {i}")
            assert (got[:2] == 0x77).all()  # nothing written before the first output


def test_empty_and_degenerate(cuda):
    import torch
    # r = 0: nothing to compute; decode with nothing erased is a no-op
    code = P.CodeSpec(4, 0, G16)
    d = torch.zeros((4, 16), dtype=torch.uint8, device=cuda)
    assert P.encode(d, code).shape == (0, 16)
    code = P.CodeSpec(4, 2, G16)
    s = torch.arange(6 * 16, dtype=torch.int32, device=cuda).to(torch.uint8).view(6, 16)
    before = s.clone()
    P.decode(s, [], code)
    assert torch.equal(s, before)
    # too many erasures / bad shapes raise like the reference
    with pytest.raises(P.PyritError) as e:
        P.decode(s, [0, 1, 2], code)
    assert e.value.code == "InsufficientShards"
    with pytest.raises(P.PyritError):
        P.encode(torch.zeros((4, 12), dtype=torch.uint8, device=cuda), code)  # 12 % 8 != 0


def test_fill_and_digest_kernels(cuda):
    import torch
    t = torch.empty(1 << 20, dtype=torch.uint8, device=cuda)
    P.fill(t, 4, 7, begin=8 * 1000, valid=8 * 1000 + 700_001)
    want = O.fill_np(4, 7, 1 << 20, valid=8 * 1000 + 700_001, begin=8 * 1000)
    np.testing.assert_array_equal(t.cpu().numpy(), want)
    d = P.digest(t, word_offset=123)
    torch.cuda.synchronize()
    assert (int(d.item()) & (2**64 - 1)) == O.digest_np(want, 123)
    # additivity over disjoint word ranges (the sharded "checksum of checksums")
    a = P.digest(t[: 1 << 19], word_offset=123)
    P.digest(t[1 << 19:], word_offset=123 + (1 << 16), out=a)
    assert int(a.item()) == int(d.item())


def test_shard_invariance_windows(cuda):
    """Encoding byte-offset shards separately == one encode (test_codec.cpp:199-212 analogue)."""
    import torch
    wl = WORKLOADS[5]
    ss = wl.fld.w * (1 << 16)
    strip = ss // wl.fld.w
    data = torch.from_numpy(seeded_symbols(wl.k, ss, wl.fld.w, 4)).to(cuda)
    whole = P.encode(data, wl.code)
    plan = P.Plan.encode(wl.code)
    for world in (2, 4, 8):
        out = torch.zeros_like(whole)
        for rank in range(world):
            lo, hi = shard(strip, rank, world)
            plan.apply([data[j].data_ptr() for j in range(wl.k)], [out[i].data_ptr() for i in range(wl.m)], strip,
                       lo, hi - lo, stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(out, whole), world


@pytest.mark.parametrize("cfg", [3, 4])
def test_host_buffer_path(cuda, cfg):
    """pyrit_encode_host / pyrit_decode_host (H2D + kernel + D2H pipeline) == device path."""
    wl = WORKLOADS[cfg]
    ss = wl.fld.w * (1 << 18)
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    L.check(L.load().pyrit_set_host_chunk(1 << 16))  # force several chunks through the slot ring
    try:
        parity = P.encode_host(data, wl.code)
        np.testing.assert_array_equal(parity, dev_encode(cuda, wl.code, data))
        if wl.op == "decode":
            full = np.concatenate([data, parity])
            work = full.copy()
            work[list(wl.erased)] = 0
            P.decode_host(work, wl.erased, wl.code)
            np.testing.assert_array_equal(work, full)
    finally:
        L.check(L.load().pyrit_set_host_chunk(0))


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_host_buffer_path_device_shards(cuda, cfg):
    """pyrit_encode_host_devices / _decode_host_devices: byte-offset shards processed
    concurrently (here 3 shards on the one visible device: the sharding and window
    arithmetic; no shard waits on another) == the single-device path."""
    import torch
    wl = WORKLOADS[cfg]
    ss = wl.fld.w * ((1 << 16) + 16 * 7)  # strip not divisible into equal 16-byte shards
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    devs = [0] * 3
    parity = P.encode_host(data, wl.code, devices=devs)
    np.testing.assert_array_equal(parity, dev_encode(cuda, wl.code, data))
    full = np.concatenate([data, parity])
    erased = list(wl.erased) or [0, 5, wl.k, wl.k + wl.m - 1]
    work = full.copy()
    work[erased] = 0
    P.decode_host(work, erased, wl.code, devices=devs)
    np.testing.assert_array_equal(work, full)
    assert torch.cuda.device_count() >= 1


@pytest.mark.parametrize("lanes", [1, 2, 4])
def test_vector_widths(cuda, lanes):
    """The 4/8/16-byte-per-thread variants of the generated kernel agree."""
    lib = L.load()
    L.check(lib.pyrit_set_lanes(lanes))
    try:
        wl = WORKLOADS[3]
        ss = wl.fld.w * 4096
        data = seeded_symbols(wl.k, ss, wl.fld.w, 2)
        np.testing.assert_array_equal(dev_encode(cuda, wl.code, data),
                                      oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data))
    finally:
        L.check(lib.pyrit_set_lanes(1))


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_kernel_modes_agree(cuda, mode, cfg):
    """Direct (LDG) and TMA-staged kernels are both bit-exact, including a partial last tile."""
    lib = L.load()
    L.check(lib.pyrit_set_kernel_mode(mode))
    try:
        wl = WORKLOADS[cfg]
        ss = wl.fld.w * (4096 + 16 * 37)  # window not a multiple of any tile
        data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
        C = P.cauchy_parity_matrix(wl.code)
        if wl.op == "encode":
            np.testing.assert_array_equal(dev_encode(cuda, wl.code, data), oracle_ring(wl.fld, C, data))
        else:
            full = np.concatenate([data, oracle_ring(wl.fld, C, data)])
            work = full.copy()
            work[list(wl.erased)] = 0
            np.testing.assert_array_equal(dev_decode(cuda, wl.code, work, wl.erased), full)
    finally:
        L.check(lib.pyrit_set_kernel_mode(0))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("mode", [0, 1])
def test_crs_baseline_kernel(cuda, cfg, mode):
    """The GPU CRS bitmatrix baseline (rep=2) is bit-exact with the ring path and the field oracle."""
    import torch
    lib = L.load()
    L.check(lib.pyrit_set_kernel_mode(mode))
    try:
        wl = WORKLOADS[cfg]
        f = wl.fld
        ss = f.w * (2048 + 16 * 5)
        data = seeded_symbols(wl.k, ss, f.w, wl.seed)
        C = P.cauchy_parity_matrix(wl.code)
        m = C if wl.op == "encode" else P.repair_matrix(wl.code, wl.erased)[2]
        src = data if wl.op == "encode" else np.concatenate([data, oracle_ring(f, C, data)])[
            P.repair_matrix(wl.code, wl.erased)[0]]
        plan = P.Plan.create(f, m, rep=P.RingRep.Crs)
        d = torch.from_numpy(np.ascontiguousarray(src)).to(cuda)
        out = torch.zeros((m.shape[0], ss), dtype=torch.uint8, device=cuda)
        plan.apply([d[j].data_ptr() for j in range(d.shape[0])], [out[i].data_ptr() for i in range(m.shape[0])],
                   ss // f.w)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), oracle_encode(f, m, src))
    finally:
        L.check(lib.pyrit_set_kernel_mode(0))


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("k,r,kind,ss", [(40, 20, 0, 4104), (40, 20, 0, 96 * 43), (20, 40, 1, 4104),
                                         (20, 40, 1, 8 * 6 * 35)])
def test_large_codes_split_rows(cuda, mode, k, r, kind, ss):
    """The paper's (60,40) and (60,20) GF(2^6) codes: rows split over thread groups
    (direct kernel) or warp groups (staged; 4/8/16-byte cp.async chunks)."""
    lib = L.load()
    L.check(lib.pyrit_set_kernel_mode(mode))
    try:
        code = P.CodeSpec(k, r, G64, P.TransformKind(kind))
        data = rand_symbols(k, ss, k * r + ss)
        C = P.cauchy_parity_matrix(code)
        par = dev_encode(cuda, code, data)
        np.testing.assert_array_equal(par, oracle_ring(G64, C, data, kind=kind))
        full = np.concatenate([data, par])
        erased = sorted(random.Random(ss).sample(range(k + r), min(k, r)))
        work = full.copy()
        work[erased] = 0
        np.testing.assert_array_equal(dev_decode(cuda, code, work, erased), full)
    finally:
        L.check(lib.pyrit_set_kernel_mode(0))


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_encode_crs_top_level(cuda, cfg):
    """encode_crs (codec.hpp:223-231) on the GPU == encode() == the field oracle."""
    import torch
    wl = WORKLOADS[cfg]
    f = wl.fld
    ss = f.w * (1024 + 16 * 3)
    data = seeded_symbols(wl.k, ss, f.w, wl.seed)
    d = torch.from_numpy(data).to(cuda)
    got = P.encode_crs(d, wl.code)
    ring = P.encode(d, wl.code)
    torch.cuda.synchronize()
    assert torch.equal(got, ring)
    np.testing.assert_array_equal(got.cpu().numpy(), oracle_encode(f, P.cauchy_parity_matrix(wl.code), data))


def test_random_codes_windows_and_batches(cuda):
    """Seeded random sweep (property style, test_schedule.cpp:104-136 generalised):
    random field, (k, r), transform, window [off, off+len), stripe batch and kernel mode;
    the device result on every window equals the oracle's ring replay of that window and
    bytes outside the window are untouched."""
    import torch
    rng = random.Random(20261020)
    fields = [G16, G64, G256, G1024, G4096]
    for case in range(40):
        f = rng.choice(fields)
        k = rng.randint(1, min(24, f.field_size() - 1))
        r = rng.randint(1, min(12, f.field_size() - k))
        kind = rng.choice([0, 0, 1])
        strip = 16 * rng.randint(1, 300) + rng.choice([0, 0, 4, 8])
        off = rng.choice([0, 4 * rng.randint(0, strip // 8)])
        length = rng.randint(1, strip - off)
        nb = rng.choice([1, 1, 3])
        mode = rng.choice([0, 1, 2])
        code = P.CodeSpec(k, r, f, P.TransformKind(kind))
        m = P.cauchy_parity_matrix(code)
        plan = P.Plan.create(f, m, P.TransformKind(kind))
        sym = f.w * strip
        data = rand_symbols(nb * k, sym, case).reshape(nb, k, sym)
        d = torch.from_numpy(data).to(cuda)
        out = torch.full((nb, r, sym), 0x77, dtype=torch.uint8, device=cuda)
        lib = L.load()
        L.check(lib.pyrit_set_kernel_mode(mode))
        try:
            plan.apply_batch([d[0, j].data_ptr() for j in range(k)], [out[0, i].data_ptr() for i in range(r)], strip,
                             nb, k * sym, r * sym, off=off, length=length,
                             stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
        finally:
            L.check(lib.pyrit_set_kernel_mode(0))
        got = out.cpu().numpy()
        for b in range(nb):
            want = np.full((r, sym), 0x77, np.uint8)
            outs = [want[i] for i in range(r)]
            O.ring_replay(O.Field(f.w, f.n, f.kind, f.s, f.r_esp, f.modulus), m, [data[b, j].copy() for j in range(k)],
                          strip, kind=kind, off=off, length=length, outs=outs)
            np.testing.assert_array_equal(got[b], want, err_msg=f"case {case}: {f} k{k} r{r} kind{kind} strip{strip} "
                                                               f"off{off} len{length} nb{nb} mode{mode} b{b}")
        plan.close()

"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU checker.

`liboracle.so` is the plain-C restatement (pyrit_oracle.c); `_ref/libpyrit_ref.so`
is the unmodified reference compiled in place from /root/reference headers by
oracle/Makefile.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm may import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libpyrit_ref.so")

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


@dataclass(frozen=True)
class Field:
    """FieldSpec (field.hpp:30-51), ring elements widened to 32 bits."""
    w: int
    n: int
    kind: int  # 0 Aop, 1 Esp
    s: int
    r_esp: int
    modulus: int


GF16 = Field(4, 5, 0, 1, 4, 0x1F)        # FieldSpec::gf16_aop (field.hpp:38-40)
GF64 = Field(6, 9, 1, 3, 2, 0x49)        # FieldSpec::gf64_esp (field.hpp:41-43)
GF256_R17 = Field(8, 17, 0, 1, 8, 0x139)  # BASELINE configs 2 and 4
GF1024 = Field(10, 11, 0, 1, 10, 0x7FF)   # BASELINE config 3
GF4096 = Field(12, 13, 0, 1, 12, 0x1FFF)  # BASELINE config 5


def build() -> None:
    """liboracle.so, and (reference tree present) _ref/libpyrit_ref.so + _ref/shim_check."""
    subprocess.run(["make", "-s", "-C", HERE, "all", "shim"], check=True)


def _load(path: str):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load(_LIB)
        _lib.or_gf_mul.restype = C.c_uint32
        _lib.or_gf_inv.restype = C.c_uint32
        _lib.or_sparse_transform.restype = C.c_uint32
        _lib.or_ring_mul.restype = C.c_uint32
        _lib.or_mix64.restype = C.c_uint64
        _lib.or_mix64.argtypes = [C.c_uint64]
        _lib.or_digest.restype = C.c_uint64
        _lib.or_digest.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        _lib.or_poly_mod.restype = C.c_uint64
        _lib.or_poly_mod.argtypes = [C.c_uint64, C.c_uint64]
        _lib.or_clmul.restype = C.c_uint64
        _lib.or_clmul.argtypes = [C.c_uint64, C.c_uint64]
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF) or os.path.isdir("/root/reference/proj/include/pyrit")


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            build()
        _ref = C.CDLL(_REF)
        for name in ("ref_gf_mul", "ref_gf_inv", "ref_ring_mul", "ref_sparse_transform", "ref_phi_E_inv"):
            getattr(_ref, name).restype = C.c_uint32
        _ref.ref_plan_create.restype = C.c_void_p
        _ref.ref_plan_create.argtypes = [C.c_uint] * 6 + [C.c_uint] * 3 + [C.c_uint64, u32p, C.c_uint]
        _ref.ref_plan_symbol.restype = C.c_void_p
        _ref.ref_plan_symbol.argtypes = [C.c_void_p, C.c_uint]
        _ref.ref_plan_run.argtypes = [C.c_void_p, C.c_uint]
        _ref.ref_plan_destroy.argtypes = [C.c_void_p]
        _ref.ref_crc32.restype = C.c_uint32
        _ref.ref_bench_point.restype = C.c_double
        _ref.ref_bench_point.argtypes = [C.c_uint] * 6 + [C.c_uint] * 5 + [C.c_uint64, C.c_uint, C.c_double]
        _ref.ref_crc32.argtypes = [C.c_char_p, C.c_uint64]
    return _ref


def _fa(f: Field):
    return (f.w, f.n, f.kind, f.s, f.r_esp, f.modulus)


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


# ---------------------------------------------------------------- oracle (C)
def gf_mul(a, b, f: Field) -> int:
    return lib().or_gf_mul(a, b, f.modulus)


def gf_inv(a, f: Field) -> int:
    return lib().or_gf_inv(a, f.w, f.modulus)


def ring_mul(a, b, f: Field) -> int:
    return lib().or_ring_mul(a, b, f.n)


def sparse_transform(u, f: Field) -> int:
    return lib().or_sparse_transform(u, f.w, f.n, f.modulus)


def fold_table(f: Field):
    out = (C.c_uint32 * 32)()
    lib().or_fold_table(f.w, f.n, f.modulus, out)
    return list(out[: f.n - f.w])


def cauchy(k, r, f: Field) -> np.ndarray:
    out = np.zeros(max(r, 1) * k, dtype=np.uint16)
    rc = lib().or_cauchy(k, r, f.w, f.modulus, out.ctypes.data_as(u16p))
    if rc:
        raise OracleError(rc)
    return out[: r * k].reshape(r, k)


def invert(m: np.ndarray, f: Field) -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.uint16)
    out = np.zeros_like(m)
    rc = lib().or_invert(m.shape[0], f.w, f.modulus, m.ctypes.data_as(u16p), out.ctypes.data_as(u16p))
    if rc:
        raise OracleError(rc)
    return out


def decode_matrix(k, r, f: Field, survivors) -> np.ndarray:
    c = cauchy(k, r, f)
    surv = np.asarray(survivors, dtype=np.uint32)
    out = np.zeros(k * k, dtype=np.uint16)
    rows = C.c_uint32(0)
    rc = lib().or_decode_matrix(k, r, f.w, f.modulus, c.ctypes.data_as(u16p), surv.ctypes.data_as(u32p),
                                out.ctypes.data_as(u16p), C.byref(rows))
    if rc:
        raise OracleError(rc)
    return out[: rows.value * k].reshape(rows.value, k)


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle error {rc}")
        self.rc = rc


def _apply(fn, f: Field, kind, m, ins, outs, strip, off, len_, extra=()):
    m = np.ascontiguousarray(m, dtype=np.uint16)
    rows, cols = m.shape
    rc = fn(f.w, f.n, f.s, f.modulus, kind, rows, cols, m.ctypes.data_as(u16p), _ptrs(ins), _ptrs(outs),
            C.c_uint64(strip), C.c_uint64(off), C.c_uint64(len_), *extra)
    if rc:
        raise OracleError(rc)


def apply_columns(f: Field, m, ins, strip, kind=0, off=0, length=None, outs=None):
    """codec.hpp:444-469 oracle_apply restated; ins: list of uint8 arrays (w*strip each)."""
    length = strip - off if length is None else length
    if outs is None:
        outs = [np.zeros(f.w * strip, dtype=np.uint8) for _ in range(np.asarray(m).shape[0])]
    _apply(lib().or_apply_columns, f, kind, m, ins, outs, strip, off, length)
    return outs


def ring_replay(f: Field, m, ins, strip, kind=0, off=0, length=None, outs=None, want_ops=False):
    """schedule.hpp:94-163 + codec.hpp:118-157 restated (ring schedule, generalized fold)."""
    length = strip - off if length is None else length
    if outs is None:
        outs = [np.zeros(f.w * strip, dtype=np.uint8) for _ in range(np.asarray(m).shape[0])]
    ops = C.c_uint64(0)
    _apply(lib().or_ring_replay, f, kind, m, ins, outs, strip, off, length, extra=(C.byref(ops),))
    return (outs, ops.value) if want_ops else outs


def decode(k, r, f: Field, symbols, erased, strip, kind=0, off=0, length=None):
    """codec.hpp:241-284 restated in place over k + r symbol arrays."""
    length = strip - off if length is None else length
    er = np.asarray(sorted(erased) if False else list(erased), dtype=np.uint32)
    rc = lib().or_decode(k, r, f.w, f.n, f.s, f.modulus, kind, _ptrs(symbols), er.ctypes.data_as(u32p),
                         len(er), C.c_uint64(strip), C.c_uint64(off), C.c_uint64(length))
    if rc:
        raise OracleError(rc)


def fill(seed, frag, length, valid=None, begin=0) -> np.ndarray:
    valid = begin + length if valid is None else valid
    out = np.empty(length, dtype=np.uint8)
    lib().or_fill(C.c_uint64(seed), C.c_uint64(frag), out.ctypes.data_as(u8p), C.c_uint64(begin),
                  C.c_uint64(length), C.c_uint64(valid))
    return out


def digest(buf: np.ndarray, word_offset=0) -> int:
    buf = np.ascontiguousarray(buf)
    return lib().or_digest(buf.ctypes.data, buf.nbytes, word_offset)


# ------------------------------------------------------- numpy restatements
_M1, _M2, _GOLD, _DG = (np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB),
                        np.uint64(0x9E3779B97F4A7C15), np.uint64(0xD6E8FEB86659FD93))


def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z + _GOLD
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def fill_np(seed, frag, length, valid=None, begin=0) -> np.ndarray:
    """Vectorised twin of or_fill (same bytes); begin and length multiples of 8."""
    valid = begin + length if valid is None else valid
    assert begin % 8 == 0 and length % 8 == 0
    q = np.arange(begin // 8, (begin + length) // 8, dtype=np.uint64)
    with np.errstate(over="ignore"):
        words = mix64_np((np.uint64(seed) << np.uint64(48)) ^ (np.uint64(frag) << np.uint64(36)) ^ q)
    out = words.view(np.uint8).copy()
    if valid < begin + length:
        out[max(valid - begin, 0):] = 0
    return out


def digest_np(buf: np.ndarray, word_offset=0) -> int:
    b = np.ascontiguousarray(buf).view(np.uint8)
    pad = (-b.nbytes) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    words = b.view(np.uint64)
    q = np.arange(word_offset, word_offset + words.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(mix64_np(words ^ (q * _DG)).sum(dtype=np.uint64))


# XorOp (schedule.hpp:42-48): 4 x uint16 + uint8 mode, 10 bytes
OP_DTYPE = np.dtype([("src_sym", "<u2"), ("src_pkt", "<u2"), ("dst_sym", "<u2"), ("dst_pkt", "<u2"),
                     ("mode", "u1")], align=True)
assert OP_DTYPE.itemsize == 10


def _ops_call(fn, *args) -> np.ndarray:
    n = C.c_uint64(0)
    rc = fn(*args, None, C.c_uint64(0), C.byref(n))
    if rc:
        raise OracleError(rc)
    ops = np.zeros(n.value, dtype=OP_DTYPE)
    rc = fn(*args, C.c_void_p(ops.ctypes.data), C.c_uint64(n.value), C.byref(n))
    if rc:
        raise OracleError(rc)
    return ops


def compile_schedule(f: Field, m, kind=0, rep=0) -> np.ndarray:
    """schedule.hpp:94-163 restated: the op list (pre, core, post) as an OP_DTYPE array."""
    m = np.ascontiguousarray(m, dtype=np.uint16)
    return _ops_call(lib().or_compile_schedule, f.w, f.n, f.s, f.modulus, kind, m.shape[0], m.shape[1],
                     m.ctypes.data_as(u16p), rep)


def compile_crs_schedule(f: Field, m) -> np.ndarray:
    """schedule.hpp:168-203 restated."""
    m = np.ascontiguousarray(m, dtype=np.uint16)
    return _ops_call(lib().or_compile_crs_schedule, f.w, f.modulus, m.shape[0], m.shape[1], m.ctypes.data_as(u16p))


def replay_ops(f: Field, k, outputs, ops, ins, outs, strip, off=0, length=None):
    """codec.hpp:118-157 restated op by op: ins[j] / outs[i] are the slot symbols (maps applied;
    the same array object twice = shared storage).  outs are updated in place."""
    length = strip - off if length is None else length
    ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
    rc = lib().or_replay_ops(f.w, f.n, k, outputs, C.c_void_p(ops.ctypes.data), C.c_uint64(len(ops)), _ptrs(ins),
                             _ptrs(outs), C.c_uint64(strip), C.c_uint64(off), C.c_uint64(length))
    if rc:
        raise OracleError(rc)
    return outs


# ----------------------------------------------------------- the reference
def ref_cauchy(k, r, f: Field) -> np.ndarray:
    out = np.zeros(max(r, 1) * k, dtype=np.uint16)
    rc = ref().ref_cauchy(k, r, f.w, f.n, f.modulus, out.ctypes.data_as(u16p))
    if rc:
        raise OracleError(rc)
    return out[: r * k].reshape(r, k)


def ref_sparse_transform(u, f: Field) -> int:
    return ref().ref_sparse_transform(u, *_fa(f))


def ref_schedule_stats(f: Field, m, transform=0, crs=0, rep=0) -> dict:
    m = np.ascontiguousarray(m, dtype=np.uint16)
    st = (C.c_uint64 * 8)()
    rc = ref().ref_schedule_stats(*_fa(f), m.shape[0], m.shape[1], m.ctypes.data_as(u16p), transform, crs,
                                  rep, st)
    if rc:
        raise OracleError(rc)
    keys = ("copy", "xor", "zero", "total", "matrix_ones", "pre", "core", "post")
    return dict(zip(keys, list(st)))


def ref_oracle_apply(f: Field, m, data: np.ndarray, symbol_size, transform=0) -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.uint16)
    out = np.zeros(m.shape[0] * symbol_size, dtype=np.uint8)
    rc = ref().ref_oracle_apply(*_fa(f), transform, m.shape[0], m.shape[1], m.ctypes.data_as(u16p),
                                data.ctypes.data_as(u8p), C.c_uint64(symbol_size), out.ctypes.data_as(u8p))
    if rc:
        raise OracleError(rc)
    return out


def ref_encode(f: Field, k, r, data: np.ndarray, symbol_size, transform=0, crs=0, threads=1) -> np.ndarray:
    out = np.zeros(r * symbol_size, dtype=np.uint8)
    rc = ref().ref_encode(*_fa(f), k, r, transform, crs, data.ctypes.data_as(u8p), C.c_uint64(symbol_size),
                          out.ctypes.data_as(u8p), threads)
    if rc:
        raise OracleError(rc)
    return out


def ref_decode(f: Field, k, r, symbols: np.ndarray, symbol_size, erased, transform=0, threads=1) -> None:
    er = np.asarray(list(erased), dtype=np.uint32)
    rc = ref().ref_decode(*_fa(f), k, r, transform, symbols.ctypes.data_as(u8p), C.c_uint64(symbol_size),
                          er.ctypes.data_as(u32p), len(er), threads)
    if rc:
        raise OracleError(rc)


def ref_schedule_ops(f: Field, m, transform=0, crs=0, rep=0) -> np.ndarray:
    """The reference's own compile_schedule / compile_crs_schedule op list (pre, core, post)."""
    m = np.ascontiguousarray(m, dtype=np.uint16)
    return _ops_call(ref().ref_schedule_ops, *_fa(f), m.shape[0], m.shape[1], m.ctypes.data_as(u16p), transform,
                     crs, rep)


def ref_replay_ops(f: Field, k, outputs, ops, inp: np.ndarray | None, in_map, out: np.ndarray, out_map,
                   symbol_size, threads=1) -> None:
    """The reference's parallel_replay (codec.hpp:176) of an op list; inp None = in and out are one
    SymbolBuffer (out).  out is updated in place."""
    ops = np.ascontiguousarray(ops, dtype=OP_DTYPE)
    im = np.asarray(in_map, dtype=np.uint32)
    om = np.asarray(out_map, dtype=np.uint32)
    same = inp is None
    src = out if same else inp
    rc = ref().ref_replay_ops(*_fa(f), k, outputs, C.c_void_p(ops.ctypes.data), C.c_uint64(len(ops)),
                              src.ctypes.data_as(u8p), src.size // symbol_size, im.ctypes.data_as(u32p),
                              out.ctypes.data_as(u8p), out.size // symbol_size, om.ctypes.data_as(u32p),
                              C.c_uint64(symbol_size), int(same), threads)
    if rc:
        raise OracleError(rc)


class RefPlan:
    """Precompiled reference schedule + preallocated SymbolBuffer (bench.hpp:146-208 method)."""

    def __init__(self, f: Field, k, r, mode, symbol_size, erased=()):
        er = np.asarray(list(erased) or [0], dtype=np.uint32)
        self.k, self.r, self.symbol_size = k, r, symbol_size
        self.h = ref().ref_plan_create(*_fa(f), k, r, mode, symbol_size, er.ctypes.data_as(u32p),
                                       len(list(erased)))
        if not self.h:
            raise OracleError(-1)

    def symbol(self, i) -> np.ndarray:
        p = ref().ref_plan_symbol(self.h, i)
        return np.ctypeslib.as_array(C.cast(p, u8p), shape=(self.symbol_size,))

    def run(self, threads=1):
        rc = ref().ref_plan_run(self.h, threads)
        if rc:
            raise OracleError(rc)

    def close(self):
        if self.h:
            ref().ref_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ------------------------------------------------ file codec (container.hpp)
# Restated in Python over the C oracle's ring_replay/decode, one stripe at a
# time exactly as the reference does (test sizes only).
HEADER_SIZE = 29  # container.hpp:38
_FIELD_IDS = {GF16: 0, GF64: 1, GF256_R17: 2, GF1024: 3, GF4096: 4}  # 0/1: field.hpp:54-62


def crc32(b: bytes) -> int:
    """container.hpp:41-55: reflected CRC-32, polynomial 0xEDB88320, init/xorout ~0."""
    c = 0xFFFFFFFF
    for x in b:
        c ^= x
        for _ in range(8):
            c = (c >> 1) ^ (0xEDB88320 if c & 1 else 0)
    return c ^ 0xFFFFFFFF


def serialize_header(field_id, transform, k, r, index, symbol_size, length) -> bytes:
    """container.hpp:114-127 (layout container.hpp:16-36, little endian)."""
    b = (b"PYRT" + bytes([1, field_id, transform]) + k.to_bytes(2, "little") + r.to_bytes(2, "little")
         + index.to_bytes(2, "little") + symbol_size.to_bytes(4, "little") + length.to_bytes(8, "little"))
    return b + crc32(b).to_bytes(4, "little")


def shard_name(input_path, index) -> str:  # container.hpp:186-189
    return f"{os.path.basename(str(input_path))}.s{index:03d}.pyrit"


def encode_file(input_path, out_dir, k, r, f: Field, symbol_size, kind=0) -> list[str]:
    """container.hpp:168-222: stripes of k symbols, zero padded, encode() per stripe."""
    data = np.fromfile(str(input_path), dtype=np.uint8)
    length = data.size
    stripe = k * symbol_size
    stripes = 0 if length == 0 else -(-length // stripe)
    padded = np.zeros(stripes * stripe, dtype=np.uint8)
    padded[:length] = data
    m = cauchy(k, r, f)
    strip = symbol_size // f.w
    payload = [[] for _ in range(k + r)]
    for s in range(stripes):
        ins = [padded[s * stripe + j * symbol_size: s * stripe + (j + 1) * symbol_size].copy() for j in range(k)]
        outs = ring_replay(f, m, ins, strip, kind) if r else []
        for j in range(k):
            payload[j].append(ins[j])
        for i in range(r):
            payload[k + i].append(outs[i])
    os.makedirs(str(out_dir), exist_ok=True)
    paths = []
    for i in range(k + r):
        p = os.path.join(str(out_dir), shard_name(input_path, i))
        with open(p, "wb") as fh:
            fh.write(serialize_header(_FIELD_IDS[f], kind, k, r, i, symbol_size, length))
            for sym in payload[i]:
                fh.write(sym.tobytes())
        paths.append(p)
    return paths


def decode_file(paths, output, k, r, f: Field, symbol_size, length, kind=0) -> None:
    """container.hpp:249-299 for a consistent set (first occurrence of an index wins)."""
    have = {}
    for p in paths:
        b = open(str(p), "rb").read()
        idx = int.from_bytes(b[11:13], "little")
        have.setdefault(idx, np.frombuffer(b[HEADER_SIZE:], dtype=np.uint8))
    stripes = 0 if length == 0 else -(-length // (k * symbol_size))
    erased = [i for i in range(k + r) if i not in have]
    out = bytearray()
    strip = symbol_size // f.w
    for s in range(stripes):
        syms = [have[i][s * symbol_size:(s + 1) * symbol_size].copy() if i in have
                else np.zeros(symbol_size, np.uint8) for i in range(k + r)]
        if erased:
            decode(k, r, f, syms, erased, strip, kind)
        for j in range(k):
            out += syms[j].tobytes()
    with open(str(output), "wb") as fh:
        fh.write(bytes(out[:length]))


def ref_encode_file(input_path, out_dir, k, r, f: Field, symbol_size, kind=0) -> None:
    rc = ref().ref_encode_file(str(input_path).encode(), str(out_dir).encode(), *_fa(f), k, r, kind,
                               C.c_uint32(symbol_size))
    if rc:
        raise OracleError(rc)


def ref_decode_file(paths, output) -> None:
    arr = (C.c_char_p * max(len(paths), 1))(*[str(p).encode() for p in paths])
    rc = ref().ref_decode_file(arr, len(paths), str(output).encode())
    if rc:
        raise OracleError(rc)


def ref_serialize_header(field_id, transform, k, r, index, symbol_size, length) -> bytes:
    out = (C.c_uint8 * HEADER_SIZE)()
    rc = ref().ref_serialize_header(field_id, transform, k, r, index, C.c_uint32(symbol_size),
                                    C.c_uint64(length), out)
    if rc:
        raise OracleError(rc)
    return bytes(out)


def ref_parse_header(b: bytes):
    buf = (C.c_uint8 * max(len(b), 1)).from_buffer_copy(b if b else b"\0")
    out = (C.c_uint64 * 8)()
    rc = ref().ref_parse_header(buf, C.c_uint64(len(b)), out)
    if rc:
        raise OracleError(rc)
    return tuple(out)


def ref_bench_point(f: Field, k, r, codec, op, size, workers, transform=0, target_seconds=0.25) -> float:
    """bench.hpp:146-208 BenchRunner::run_point (GB/s, (k + r) * size convention); w <= 6 only."""
    return ref().ref_bench_point(*_fa(f), k, r, transform, codec, op, size, workers, target_seconds)

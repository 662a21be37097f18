"""B200-native PYRIT ring codec -- Python mirror of the reference C++ API.

Names, argument meaning and errors follow the reference library
(/root/reference/proj/include/pyrit/, cited per function); the work is done
by libpyrit_b200.so (C++ host algebra + generated sm_100a kernels) through the
C ABI in include/pyrit_b200.h.  Device entry points take CUDA torch tensors;
host entry points take numpy arrays laid out like SymbolBuffer
(codec.hpp:24-73: symbols contiguous, each w strips of symbol_size/w bytes).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L
from ._lib import PyritError

__all__ = [
    "FieldSpec", "CodeSpec", "TransformKind", "RingRep", "PyritError", "Plan", "gf_mul", "gf_inv",
    "sparse_transform", "fold_table", "cauchy_parity_matrix", "decode_matrix", "repair_matrix", "encode",
    "decode", "encode_host", "decode_host", "fill", "digest", "choose_transform", "encode_batch", "decode_batch",
    "ShardHeader", "crc32", "serialize_header", "parse_header", "field_id", "field_from_id", "shard_path",
    "encode_file", "decode_file", "HEADER_SIZE", "encode_crs", "XorSchedule", "OP_DTYPE", "replay",
    "parallel_replay",
]


class TransformKind(enum.IntEnum):  # transform.hpp:24
    Embedding = 0
    Parity = 1


class RingRep(enum.IntEnum):  # schedule.hpp:78
    Sparse = 0
    Dense = 1
    Crs = 2  # not a ring representative: the bitmatrix program of compile_crs_schedule (schedule.hpp:168-203)


def choose_transform(k: int, r: int) -> TransformKind:  # schedule.hpp:71-73
    return TransformKind.Embedding if k >= r else TransformKind.Parity


@dataclass(frozen=True)
class FieldSpec:
    """field.hpp:30-51; ring elements are 32-bit so R_{2,17} is representable."""
    w: int
    n: int
    kind: int = 0
    s: int = 1
    r_esp: int = 0
    modulus: int = 0

    @staticmethod
    def gf16_aop() -> "FieldSpec":  # field.hpp:38-40
        return FieldSpec(4, 5, 0, 1, 4, 0b11111)

    @staticmethod
    def gf64_esp() -> "FieldSpec":  # field.hpp:41-43
        return FieldSpec(6, 9, 1, 3, 2, 0b001001001)

    @staticmethod
    def gf256_r17() -> "FieldSpec":  # BASELINE configs 2/4: p = x^8+x^5+x^4+x^3+1 | x^17+1
        return FieldSpec(8, 17, 0, 1, 8, 0x139)

    @staticmethod
    def aop(w: int) -> "FieldSpec":  # all-one p of degree w in R_{2,w+1} (field.hpp:103-132)
        return FieldSpec(w, w + 1, 0, 1, w, (1 << (w + 1)) - 1)

    def c(self) -> L.pyrit_field:
        return L.pyrit_field(self.w, self.n, self.kind, self.s, self.r_esp or self.w, self.modulus)

    def field_size(self) -> int:
        return 1 << self.w


@dataclass(frozen=True)
class CodeSpec:
    """matrix.hpp:16-23."""
    k: int
    r: int
    field: FieldSpec
    transform: TransformKind = TransformKind.Embedding

    def c(self) -> L.pyrit_code:
        return L.pyrit_code(self.k, self.r, self.field.c(), int(self.transform))


def _clib():
    return L.load()


def _u32(x) -> C.c_uint32:
    return C.c_uint32(x)


def gf_mul(a: int, b: int, f: FieldSpec) -> int:  # field.hpp:68
    out = C.c_uint32()
    L.check(_clib().pyrit_gf_mul(C.byref(f.c()), a, b, C.byref(out)))
    return out.value


def gf_inv(a: int, f: FieldSpec) -> int:  # field.hpp:82
    out = C.c_uint32()
    L.check(_clib().pyrit_gf_inv(C.byref(f.c()), a, C.byref(out)))
    return out.value


def sparse_transform(u: int, f: FieldSpec) -> int:  # ring.hpp:77
    out = C.c_uint32()
    L.check(_clib().pyrit_sparse_transform(C.byref(f.c()), u, C.byref(out)))
    return out.value


def fold_table(f: FieldSpec) -> list[int]:
    out = (C.c_uint32 * 32)()
    L.check(_clib().pyrit_fold_table(C.byref(f.c()), out))
    return list(out[: f.n - f.w])


def cauchy_parity_matrix(code: CodeSpec) -> np.ndarray:  # matrix.hpp:54-80
    out = np.zeros(max(code.r * code.k, 1), dtype=np.uint16)
    L.check(_clib().pyrit_cauchy_parity_matrix(C.byref(code.c()), out.ctypes.data))
    return out[: code.r * code.k].reshape(code.r, code.k)


def decode_matrix(code: CodeSpec, survivors: Sequence[int]) -> np.ndarray:  # matrix.hpp:193-220
    surv = np.asarray(survivors, dtype=np.uint32)
    if surv.size != code.k:
        raise PyritError(11, "need exactly k survivors")
    out = np.zeros(code.k * code.k, dtype=np.uint16)
    rows = C.c_uint32()
    L.check(_clib().pyrit_decode_matrix(C.byref(code.c()), surv.ctypes.data, out.ctypes.data, C.byref(rows)))
    return out[: rows.value * code.k].reshape(rows.value, code.k)


def repair_matrix(code: CodeSpec, erased: Iterable[int]):
    """Fused one-pass repair: (survivors, outputs, matrix over survivors)."""
    er = np.asarray(list(erased), dtype=np.uint32)
    surv = np.zeros(code.k, dtype=np.uint32)
    outs = np.zeros(max(er.size, 1), dtype=np.uint32)
    m = np.zeros(max(er.size, 1) * code.k, dtype=np.uint16)
    L.check(_clib().pyrit_repair_matrix(C.byref(code.c()), er.ctypes.data, er.size, surv.ctypes.data,
                                       outs.ctypes.data, m.ctypes.data))
    return surv, outs[: er.size], m[: er.size * code.k].reshape(er.size, code.k)


# XorOp (schedule.hpp:42-48): src_sym, src_pkt, dst_sym, dst_pkt (uint16), mode (OpMode, uint8:
# 0 Copy, 1 Xor, 2 Zero) -- 10 bytes, the reference's own layout
OP_DTYPE = np.dtype([("src_sym", "<u2"), ("src_pkt", "<u2"), ("dst_sym", "<u2"), ("dst_pkt", "<u2"),
                     ("mode", "u1")], align=True)


@dataclass
class XorSchedule:
    """schedule.hpp:50-58: k input slots, `outputs` output slots, and the region ops of the pre, core
    and post phases concatenated in replay order (an OP_DTYPE array)."""
    spec: FieldSpec
    k: int
    outputs: int
    ops: np.ndarray

    def __post_init__(self):
        self.ops = np.ascontiguousarray(self.ops, dtype=OP_DTYPE)


def jit_info() -> str:
    """Which NVRTC compiles kernels that are not prebuilt, e.g. 'nvrtc 12.9 (/usr/local/cuda/lib64/libnvrtc.so.12)'."""
    buf = C.create_string_buffer(512)
    L.check(_clib().pyrit_jit_info(buf, 512))
    return buf.value.decode()


def _ptr_array(ptrs):
    return (C.c_void_p * max(len(ptrs), 1))(*ptrs)


class Plan:
    """A compiled ring program: the GPU counterpart of XorSchedule (schedule.hpp:50-59)."""

    def __init__(self, handle: C.c_void_p, survivors=None, outputs=None, shape=None):
        self._h = handle
        self.slots = None
        self.survivors = survivors
        self.outputs = outputs
        self._shape = shape  # (rows, cols) when known at creation: no compile needed to check calls

    @classmethod
    def create(cls, f: FieldSpec, matrix: np.ndarray, transform=TransformKind.Embedding, rep=RingRep.Sparse,
               group: int = 0) -> "Plan":  # compile_schedule(m, kind, rep), schedule.hpp:94
        m = np.ascontiguousarray(matrix, dtype=np.uint16)
        h = C.c_void_p()
        L.check(_clib().pyrit_plan_create(C.byref(f.c()), int(transform), m.ctypes.data, m.shape[0], m.shape[1],
                                         int(rep), group, C.byref(h)))
        return cls(h, shape=m.shape)

    @classmethod
    def from_ringmat(cls, f: FieldSpec, reps: np.ndarray, transform=TransformKind.Embedding) -> "Plan":
        """A plan of raw ring representatives (n-bit shift masks, any element of each coset;
        SURVEY 8(b) pyrit_cu_ringmat): runs on the runtime-matrix kernel, never compiled."""
        r = np.ascontiguousarray(reps, dtype=np.uint32)
        m = L.pyrit_ringmat(f.c(), int(transform), r.shape[0], r.shape[1], r.ctypes.data)
        h = C.c_void_p()
        L.check(_clib().pyrit_plan_from_ringmat(C.byref(m), C.byref(h)))
        return cls(h, shape=r.shape)

    @classmethod
    def from_schedule(cls, sched: XorSchedule, labels: Sequence[int] | None = None) -> "Plan":
        """Any XorSchedule as one fused kernel with replay()'s semantics (codec.hpp:118-157); labels:
        k + outputs storage labels, equal labels = slots sharing storage (None = all distinct)."""
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint32)
        h = C.c_void_p()
        L.check(_clib().pyrit_plan_from_schedule(C.byref(sched.spec.c()), sched.k, sched.outputs,
                                                sched.ops.ctypes.data, len(sched.ops),
                                                None if lab is None else lab.ctypes.data, C.byref(h)))
        plan = cls(h)
        plan.slots = (sched.k, sched.outputs)  # in[] / out[] are indexed by slot for these plans
        return plan

    @classmethod
    def encode(cls, code: CodeSpec) -> "Plan":
        h = C.c_void_p()
        L.check(_clib().pyrit_plan_encode(C.byref(code.c()), C.byref(h)))
        return cls(h, shape=(code.r, code.k))

    @classmethod
    def decode(cls, code: CodeSpec, erased: Iterable[int]) -> "Plan":
        er = np.asarray(list(erased), dtype=np.uint32)
        surv = np.zeros(code.k, dtype=np.uint32)
        outs = np.zeros(max(er.size, 1), dtype=np.uint32)
        h = C.c_void_p()
        L.check(_clib().pyrit_plan_decode(C.byref(code.c()), er.ctypes.data, er.size, C.byref(h), surv.ctypes.data,
                                         outs.ctypes.data))
        return cls(h, surv.tolist(), outs[: er.size].tolist(), shape=(int(er.size), code.k))

    def stats(self) -> dict:
        st = L.pyrit_plan_stats()
        L.check(_clib().pyrit_plan_get_stats(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in L.pyrit_plan_stats._fields_}

    def key(self) -> str:
        """Tuning-table key (field, transform, ring representatives)."""
        buf = C.create_string_buffer(96)
        L.check(_clib().pyrit_plan_key(self._h, buf, 96))
        return buf.value.decode()

    def reps(self) -> np.ndarray:
        st = self.stats()
        out = np.zeros(st["rows"] * st["cols"], dtype=np.uint32)
        L.check(_clib().pyrit_plan_reps(self._h, out.ctypes.data))
        return out.reshape(st["rows"], st["cols"])

    def source(self, lanes: int = 1) -> tuple[str, str]:
        size = C.c_size_t()
        name = C.create_string_buffer(128)
        L.check(_clib().pyrit_plan_source(self._h, lanes, None, 0, C.byref(size), name, 128))
        buf = C.create_string_buffer(size.value + 1)
        L.check(_clib().pyrit_plan_source(self._h, lanes, buf, size.value + 1, None, None, 0))
        return name.value.decode(), buf.value.decode()

    def interpret(self, ins: Sequence[np.ndarray], strip: int, off: int = 0, length: int | None = None,
                  outs: Sequence[np.ndarray] | None = None) -> list[np.ndarray]:
        """Run the compiled program on host arrays (compiler verification only)."""
        st = self.stats()
        length = strip - off if length is None else length
        n_in, n_out = getattr(self, "slots", None) or (st["cols"], st["rows"])
        if len(ins) < n_in:
            raise PyritError(4, f"{n_in} input symbols expected")
        if outs is None:
            outs = [np.zeros(len(ins[0]), dtype=np.uint8) for _ in range(n_out)]
        if len(outs) < n_out:
            raise PyritError(4, f"{n_out} output symbols expected")
        L.check(_clib().pyrit_plan_interpret(self._h, _ptr_array([a.ctypes.data for a in ins]),
                                            _ptr_array([a.ctypes.data for a in outs]), strip, off, length))
        return list(outs)

    def interpret_rt(self, in_ptrs: Sequence[int], out_ptrs: Sequence[int], strip: int, off: int = 0,
                     length: int | None = None, stripes: int = 1, in_pitch: int = 0, out_pitch: int = 0) -> None:
        """The runtime-matrix kernel's launch plan run on HOST memory (pointers to 16-byte
        aligned host buffers; verification of the planner only)."""
        self._counts(in_ptrs, out_ptrs)
        length = strip - off if length is None else length
        L.check(_clib().pyrit_rt_interpret(self._h, _ptr_array(in_ptrs), _ptr_array(out_ptrs), strip, off, length,
                                           stripes, in_pitch, out_pitch))

    def rt_info(self) -> dict:
        """How the runtime-matrix planner runs this plan (host only): launches, ring terms,
        ops (a paired-shift op covers two terms) and bytes of dispatch-case code named."""
        info = (C.c_uint32 * 4)()
        L.check(_clib().pyrit_rt_plan_info(self._h, info))
        return {"launches": info[0], "terms": info[1], "ops": info[2], "case_bytes": info[3]}

    def _counts(self, ins, outs) -> None:
        """The C ABI reads in[]/out[] by slot count: refuse short pointer lists here."""
        if self.slots is None:
            if self._shape is not None:  # known at creation (stats() would compile a light plan)
                n_out, n_in = int(self._shape[0]), int(self._shape[1])
            else:
                st = self.stats()
                n_in, n_out = st["cols"], st["rows"]
        else:
            n_in, n_out = self.slots
        if len(ins) < n_in or len(outs) < n_out:
            raise PyritError(4, f"{n_in} input and {n_out} output symbols expected")

    def apply(self, in_ptrs: Sequence[int], out_ptrs: Sequence[int], strip: int, off: int = 0,
              length: int | None = None, stream: int | None = None) -> None:
        """replay (codec.hpp:118) over device pointers, asynchronously on `stream`."""
        self._counts(in_ptrs, out_ptrs)
        length = strip - off if length is None else length
        L.check(_clib().pyrit_cu_apply(self._h, _ptr_array(list(in_ptrs)), _ptr_array(list(out_ptrs)), strip, off,
                                      length, stream))

    def apply_host(self, ins: Sequence[np.ndarray], outs: Sequence[np.ndarray], strip: int, off: int = 0,
                   length: int | None = None, device: int = 0) -> None:
        """replay over HOST symbols (numpy uint8, w strips each): H2D, kernel, D2H inside; synchronous."""
        self._counts(ins, outs)
        length = strip - off if length is None else length
        L.check(_clib().pyrit_apply_host(self._h, _ptr_array([a.ctypes.data for a in ins]),
                                        _ptr_array([a.ctypes.data for a in outs]), strip, off, length, device))

    @staticmethod
    def last_launch() -> dict:
        """Kernel name / grid of this thread's most recent launch through the C ABI."""
        name = C.create_string_buffer(128)
        blocks, threads = C.c_uint32(), C.c_uint32()
        L.check(_clib().pyrit_cu_last_launch(name, 128, C.byref(blocks), C.byref(threads)))
        return {"kernel": name.value.decode(), "blocks": blocks.value, "threads": threads.value}

    def apply_batch(self, in_ptrs: Sequence[int], out_ptrs: Sequence[int], strip: int, stripes: int,
                    in_pitch: int, out_pitch: int, off: int = 0, length: int | None = None,
                    stream: int | None = None) -> None:
        """`stripes` stripes in one launch: input j of stripe b at in_ptrs[j] + b * in_pitch."""
        self._counts(in_ptrs, out_ptrs)
        length = strip - off if length is None else length
        L.check(_clib().pyrit_cu_apply_batch(self._h, _ptr_array(list(in_ptrs)), _ptr_array(list(out_ptrs)), strip,
                                            off, length, stripes, in_pitch, out_pitch, stream))

    def inject_fault(self, entry: int, bit: int) -> None:
        """Negative control (tools/pyrit.cpp:281-282 --inject-theta-fault): flip bit `bit` of the ring
        representative of matrix entry `entry` and recompile; the plan is then WRONG on purpose."""
        L.check(_clib().pyrit_plan_inject_fault(self._h, entry, bit))

    def prepare(self) -> None:
        L.check(_clib().pyrit_cu_prepare(self._h))

    def close(self):
        if self._h:
            _clib().pyrit_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_of(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _rows(t) -> list[int]:
    return [t[i].data_ptr() for i in range(t.shape[0])]


def _replay_checks(sched: XorSchedule, inp, in_map, out, out_map, offset, length):
    # codec.hpp:122-127
    if len(in_map) != sched.k or len(out_map) != sched.outputs:
        raise PyritError(4, "replay: slot map sizes do not match schedule")
    if inp.shape[1] != out.shape[1] or inp.shape[1] % sched.spec.w:
        raise PyritError(4, "replay: field mismatch")
    for t in (inp, out):  # every symbol's strips must be contiguous bytes (SymbolBuffer layout)
        unit = t.stride(1) if hasattr(t, "stride") and callable(t.stride) else t.strides[1]
        if unit != 1 or str(t.dtype) not in ("torch.uint8", "uint8"):
            raise PyritError(4, "replay: symbols must be uint8 rows with contiguous bytes")
    strip = inp.shape[1] // sched.spec.w
    length = strip - offset if length is None else length
    if offset + length > strip:
        raise PyritError(4, "replay: column window out of range")
    for j in in_map:
        if not 0 <= j < inp.shape[0]:
            raise PyritError(4, "replay: input slot maps outside the buffer")
    for i in out_map:
        if not 0 <= i < out.shape[0]:
            raise PyritError(4, "replay: output slot maps outside the buffer")
    return strip, length


def replay(sched: XorSchedule, inp, in_map: Sequence[int], out, out_map: Sequence[int], offset: int = 0,
           length: int | None = None, device: int = 0) -> None:
    """replay (codec.hpp:118-157) of any schedule over the column window [offset, offset+length) of every
    packet, on the GPU: `inp` / `out` are (symbols, symbol_size) uint8 CUDA tensors (asynchronous on the
    current stream) or numpy arrays (host path, synchronous); they may be the same buffer (decode() style).
    Workspace scratch starts zeroed, as in parallel_replay."""
    strip, length = _replay_checks(sched, inp, in_map, out, out_map, offset, length)
    if hasattr(inp, "data_ptr"):
        ins = [inp[j].data_ptr() for j in in_map]
        outs = [out[i].data_ptr() for i in out_map]
    else:
        ins = [inp[j].ctypes.data for j in in_map]
        outs = [out[i].ctypes.data for i in out_map]
    addr = ins + outs  # slots sharing a symbol share storage
    labels = [addr.index(a) for a in addr]
    plan = Plan.from_schedule(sched, labels)
    if hasattr(inp, "data_ptr"):
        L.check(_clib().pyrit_cu_apply(plan._h, _ptr_array(ins), _ptr_array(outs), strip, offset, length,
                                      _stream_of(out)))
    else:
        L.check(_clib().pyrit_apply_host(plan._h, _ptr_array(ins), _ptr_array(outs), strip, offset, length, device))


def parallel_replay(sched: XorSchedule, inp, in_map: Sequence[int], out, out_map: Sequence[int],
                    device: int = 0) -> None:
    """parallel_replay (codec.hpp:176-193): replay over the whole packet (the column windows of the
    reference's threads are one grid here)."""
    replay(sched, inp, in_map, out, out_map, 0, None, device)


def apply_ringmat(f: FieldSpec, reps: np.ndarray, in_ptrs: Sequence[int], out_ptrs: Sequence[int], strip: int,
                  off: int = 0, length: int | None = None, transform=TransformKind.Embedding,
                  stream: int | None = None) -> None:
    """out[i] = sum_j reps[i][j] * in[j] on device pointers (pyrit_cu_apply_ringmat): the
    runtime-matrix kernel with the masks in its parameters, asynchronously on `stream`."""
    r = np.ascontiguousarray(reps, dtype=np.uint32)
    if len(in_ptrs) < r.shape[1] or len(out_ptrs) < r.shape[0]:
        raise PyritError(4, f"{r.shape[1]} input and {r.shape[0]} output symbols expected")
    length = strip - off if length is None else length
    m = L.pyrit_ringmat(f.c(), int(transform), r.shape[0], r.shape[1], r.ctypes.data)
    L.check(_clib().pyrit_cu_apply_ringmat(C.byref(m), _ptr_array(in_ptrs), _ptr_array(out_ptrs), strip, off, length,
                                           stream))


def encode(data, code: CodeSpec):
    """encode (codec.hpp:212-220): data is a (k, symbol_size) uint8 CUDA tensor; returns (r, symbol_size)."""
    import torch
    if data.dim() != 2 or data.shape[0] != code.k or data.dtype != torch.uint8 or not data.is_cuda:
        raise PyritError(4, "data buffer does not match the code")
    data = data.contiguous()
    parity = torch.empty((code.r, data.shape[1]), dtype=torch.uint8, device=data.device)
    L.check(_clib().pyrit_cu_encode(C.byref(code.c()), _ptr_array(_rows(data)), _ptr_array(_rows(parity)),
                                   data.shape[1], _stream_of(data)))
    return parity


def encode_crs(data, code: CodeSpec):
    """encode_crs (codec.hpp:223-231): the Cauchy-RS bitmatrix baseline on the GPU; same parity bytes."""
    import torch
    if data.dim() != 2 or data.shape[0] != code.k or data.dtype != torch.uint8 or not data.is_cuda:
        raise PyritError(4, "data buffer does not match the code")
    data = data.contiguous()
    parity = torch.empty((code.r, data.shape[1]), dtype=torch.uint8, device=data.device)
    L.check(_clib().pyrit_cu_encode_crs(C.byref(code.c()), _ptr_array(_rows(data)), _ptr_array(_rows(parity)),
                                       data.shape[1], _stream_of(data)))
    return parity


def decode(symbols, erased: Iterable[int], code: CodeSpec) -> None:
    """decode (codec.hpp:241-284), in place on a (k + r, symbol_size) uint8 CUDA tensor."""
    import torch
    if symbols.dim() != 2 or symbols.shape[0] != code.k + code.r or symbols.dtype != torch.uint8:
        raise PyritError(4, "symbol buffer does not match the code")
    if not symbols.is_cuda or symbols.stride(1) != 1:
        raise PyritError(4, "symbols must be CUDA rows with contiguous bytes (repaired in place)")
    er = np.asarray(list(erased), dtype=np.uint32)
    L.check(_clib().pyrit_cu_decode(C.byref(code.c()), _ptr_array(_rows(symbols)), er.ctypes.data, er.size,
                                   symbols.shape[1], _stream_of(symbols)))


def encode_host(data: np.ndarray, code: CodeSpec, device: int = 0, parity: np.ndarray | None = None,
                devices: Sequence[int] | None = None) -> np.ndarray:
    """encode with host buffers (H2D, fused kernel, D2H inside): data (k, symbol_size) uint8.
    `devices`: byte-offset shards over several GPUs, concurrently."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.ndim != 2 or data.shape[0] != code.k:
        raise PyritError(4, "data buffer does not match the code")
    if parity is None:
        parity = np.empty((code.r, data.shape[1]), dtype=np.uint8)
    elif parity.shape != (code.r, data.shape[1]) or parity.dtype != np.uint8 or not parity.flags.c_contiguous:
        raise PyritError(4, "parity buffer does not match the code")
    if devices:
        dv = np.asarray(list(devices), dtype=np.int32)
        L.check(_clib().pyrit_encode_host_devices(C.byref(code.c()), data.ctypes.data, parity.ctypes.data,
                                                 data.shape[1], dv.ctypes.data, dv.size))
    else:
        L.check(_clib().pyrit_encode_host(C.byref(code.c()), data.ctypes.data, parity.ctypes.data, data.shape[1],
                                         device))
    return parity


def decode_host(symbols: np.ndarray, erased: Iterable[int], code: CodeSpec, device: int = 0,
                devices: Sequence[int] | None = None) -> None:
    """decode with host buffers, in place on a (k + r, symbol_size) uint8 array."""
    if symbols.ndim != 2 or symbols.shape[0] != code.k + code.r or not symbols.flags.c_contiguous:
        raise PyritError(4, "symbol buffer does not match the code")
    er = np.asarray(list(erased), dtype=np.uint32)
    if devices:
        dv = np.asarray(list(devices), dtype=np.int32)
        L.check(_clib().pyrit_decode_host_devices(C.byref(code.c()), symbols.ctypes.data, er.ctypes.data, er.size,
                                                 symbols.shape[1], dv.ctypes.data, dv.size))
    else:
        L.check(_clib().pyrit_decode_host(C.byref(code.c()), symbols.ctypes.data, er.ctypes.data, er.size,
                                         symbols.shape[1], device))


def fill(t, seed: int, frag: int, begin: int = 0, valid: int | None = None, stream: int | None = None) -> None:
    """Seeded synthetic bytes (same definition as oracle/pyrit_oracle.c or_fill) into a CUDA tensor."""
    n = t.numel()
    valid = begin + n if valid is None else valid
    L.check(_clib().pyrit_cu_fill(seed, frag, t.data_ptr(), begin, n, valid,
                                 _stream_of(t) if stream is None else stream))


def digest(t, word_offset: int = 0, out=None, stream: int | None = None):
    """K3 slice digest: out (1-element uint64 CUDA tensor) += digest(t)."""
    import torch
    if out is None:
        out = torch.zeros(1, dtype=torch.int64, device=t.device)
    L.check(_clib().pyrit_cu_digest(t.data_ptr(), t.numel(), word_offset, out.data_ptr(),
                                   _stream_of(t) if stream is None else stream))
    return out


def encode_batch(data, code: CodeSpec, symbol_size: int):
    """Stripe batch encode: data is a (stripes, k * symbol_size) uint8 CUDA tensor laid out
    like the input file of encode_file (container.hpp:204-212: stripe = k symbols);
    returns parity (r, stripes, symbol_size) -- shard order, one launch for all stripes."""
    import torch
    if data.dim() != 2 or data.shape[1] != code.k * symbol_size or data.dtype != torch.uint8 or not data.is_cuda:
        raise PyritError(4, "data buffer does not match the code")
    data = data.contiguous()
    nb = data.shape[0]
    parity = torch.empty((code.r, nb, symbol_size), dtype=torch.uint8, device=data.device)
    base = data.data_ptr()
    ins = [base + j * symbol_size for j in range(code.k)]
    outs = [parity[i].data_ptr() for i in range(code.r)]
    L.check(_clib().pyrit_cu_encode_batch(C.byref(code.c()), _ptr_array(ins), _ptr_array(outs), symbol_size, nb,
                                         code.k * symbol_size, symbol_size, _stream_of(data)))
    return parity


def decode_batch(symbols, erased: Iterable[int], code: CodeSpec) -> None:
    """Stripe batch repair in place: symbols is a (k + r, stripes, symbol_size) uint8 CUDA tensor."""
    import torch
    if symbols.dim() != 3 or symbols.shape[0] != code.k + code.r or symbols.dtype != torch.uint8:
        raise PyritError(4, "symbol buffer does not match the code")
    if not symbols.is_contiguous():
        raise PyritError(4, "symbol buffer must be contiguous")
    er = np.asarray(list(erased), dtype=np.uint32)
    ss = symbols.shape[2]
    L.check(_clib().pyrit_cu_decode_batch(C.byref(code.c()), _ptr_array(_rows(symbols)), er.ctypes.data, er.size,
                                         ss, symbols.shape[1], ss, _stream_of(symbols)))


# ---- shard container (container.hpp) -------------------------------------

HEADER_SIZE = L.HEADER_SIZE


@dataclass(frozen=True)
class ShardHeader:
    """container.hpp:57-84."""
    version: int = 1
    field: int = 0
    transform: int = 0
    k: int = 0
    r: int = 0
    shard_index: int = 0
    symbol_size: int = 0
    original_length: int = 0

    def same_set(self, o: "ShardHeader") -> bool:  # container.hpp:70-74
        return (self.version, self.field, self.transform, self.k, self.r, self.symbol_size,
                self.original_length) == (o.version, o.field, o.transform, o.k, o.r, o.symbol_size,
                                          o.original_length)

    def stripe_count(self) -> int:  # container.hpp:80-83
        sb = self.k * self.symbol_size
        return 0 if sb == 0 else (self.original_length + sb - 1) // sb


def crc32(data: bytes) -> int:  # container.hpp:41-55
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    return int(_clib().pyrit_crc32(buf.ctypes.data if buf.size else None, buf.size))


def serialize_header(h: ShardHeader) -> bytes:  # container.hpp:114-127
    out = (C.c_uint8 * HEADER_SIZE)()
    ch = L.pyrit_shard_header(h.version, h.field, h.transform, h.k, h.r, h.shard_index, h.symbol_size,
                              h.original_length)
    L.check(_clib().pyrit_header_serialize(C.byref(ch), out))
    return bytes(out)


def parse_header(data: bytes) -> ShardHeader:  # container.hpp:132-161
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    ch = L.pyrit_shard_header()
    L.check(_clib().pyrit_header_parse(buf.ctypes.data if buf.size else None, buf.size, C.byref(ch)))
    return ShardHeader(*(getattr(ch, k) for k, _ in L.pyrit_shard_header._fields_))


def field_id(f: FieldSpec) -> int:  # field.hpp:54-56 (+ ids 2..4 for the BASELINE fields)
    out = C.c_uint8()
    L.check(_clib().pyrit_field_id(C.byref(f.c()), C.byref(out)))
    return out.value


def field_from_id(i: int) -> FieldSpec:  # field.hpp:58-62
    out = L.pyrit_field()
    L.check(_clib().pyrit_field_from_id(i, C.byref(out)))
    return FieldSpec(out.w, out.n, out.kind, out.s, out.r_esp, out.modulus)


def shard_path(input_path: str, out_dir: str, index: int) -> str:  # container.hpp:186-189
    buf = C.create_string_buffer(4096)
    L.check(_clib().pyrit_shard_path(str(input_path).encode(), str(out_dir).encode(), index, buf, 4096))
    return buf.value.decode()


def encode_file(input_path, out_dir, code: CodeSpec, symbol_size: int, device: int = 0) -> list[str]:
    """encode_file (container.hpp:168-222) through the GPU; returns the shard paths in index order."""
    L.check(_clib().pyrit_encode_file(C.byref(code.c()), str(input_path).encode(), str(out_dir).encode(),
                                     symbol_size, device))
    return [shard_path(input_path, out_dir, i) for i in range(code.k + code.r)]


def decode_file(shard_paths: Sequence, output, device: int = 0) -> None:
    """decode_file (container.hpp:249-299) through the GPU."""
    arr = (C.c_char_p * max(len(shard_paths), 1))(*[str(p).encode() for p in shard_paths])
    L.check(_clib().pyrit_decode_file(arr, len(shard_paths), str(output).encode(), device))

"""ctypes binding of libpyrit_b200.so (include/pyrit_b200.h).

The library is built in-tree by `python -m paper_1709_00178_b200.build`.  There
is no fallback: if the shared object is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libpyrit_b200.so")

ERRC = ("ZeroInverse", "Singular", "TooManySymbols", "BufferShape", "TransformMismatch", "InsufficientShards",
        "HeaderMismatch", "ChecksumError", "BadHeader", "IoError", "InvalidArgument")


class pyrit_field(C.Structure):
    _fields_ = [("w", C.c_uint32), ("n", C.c_uint32), ("kind", C.c_uint32), ("s", C.c_uint32),
                ("r_esp", C.c_uint32), ("modulus", C.c_uint32)]


class pyrit_code(C.Structure):
    _fields_ = [("k", C.c_uint32), ("r", C.c_uint32), ("field", pyrit_field), ("transform", C.c_uint32)]


class pyrit_ringmat(C.Structure):
    _fields_ = [("field", pyrit_field), ("transform", C.c_uint32), ("rows", C.c_uint32), ("cols", C.c_uint32),
                ("reps", C.c_void_p)]


class pyrit_plan_stats(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("matrix_ones", C.c_uint64),
                ("ref_region_ops", C.c_uint64), ("naive_xors", C.c_uint64), ("xors", C.c_uint64),
                ("loads", C.c_uint64), ("stores", C.c_uint64), ("group", C.c_uint32), ("parts", C.c_uint32),
                ("part_xors", C.c_uint64)]


SOURCE_STAGED = 100


class PyritError(RuntimeError):
    """Mirror of pyrit::Error (errors.hpp:26-35): carries the Errc name/code."""

    def __init__(self, rc: int, msg: str):
        self.rc = rc
        self.code = ERRC[rc - 1] if 1 <= rc <= len(ERRC) else "CudaError"
        super().__init__(f"{self.code} ({rc}): {msg}")


_lib = None

EXPORTS = (
    "pyrit_version", "pyrit_strerror", "pyrit_field_named", "pyrit_field_validate", "pyrit_gf_mul", "pyrit_gf_inv",
    "pyrit_sparse_transform", "pyrit_fold_table", "pyrit_cauchy_parity_matrix", "pyrit_decode_matrix",
    "pyrit_repair_matrix", "pyrit_plan_create", "pyrit_plan_encode", "pyrit_plan_decode", "pyrit_plan_get_stats",
    "pyrit_plan_reps", "pyrit_plan_inject_fault", "pyrit_plan_key", "pyrit_plan_source", "pyrit_plan_interpret", "pyrit_plan_destroy", "pyrit_cu_apply",
    "pyrit_cu_prepare", "pyrit_cu_encode", "pyrit_cu_decode", "pyrit_encode_host", "pyrit_decode_host",
    "pyrit_set_host_chunk", "pyrit_cu_fill", "pyrit_cu_digest", "pyrit_set_lanes", "pyrit_set_kernel_mode", "pyrit_set_kernel_dir",
    "pyrit_cu_last_launch", "pyrit_jit_compiles", "pyrit_kernel_launches", "pyrit_cu_apply_batch",
    "pyrit_cu_encode_batch", "pyrit_cu_decode_batch", "pyrit_crc32", "pyrit_header_serialize", "pyrit_header_parse",
    "pyrit_field_id", "pyrit_field_from_id", "pyrit_shard_path", "pyrit_encode_file", "pyrit_decode_file",
    "pyrit_set_file_chunk", "pyrit_cu_encode_crs", "pyrit_encode_crs_host", "pyrit_encode_host_devices",
    "pyrit_decode_host_devices", "pyrit_plan_from_schedule", "pyrit_apply_host", "pyrit_jit_info",
    "pyrit_jit_wait", "pyrit_jit_time", "pyrit_rt_interpret", "pyrit_plan_from_ringmat", "pyrit_cu_apply_ringmat",
    "pyrit_warmup", "pyrit_rt_plan_info", "pyrit_numa_bind_thread", "pyrit_bind_thread_cpulist",
)

HEADER_SIZE = 29


class pyrit_shard_header(C.Structure):
    _fields_ = [("version", C.c_uint8), ("field", C.c_uint8), ("transform", C.c_uint8), ("k", C.c_uint16),
                ("r", C.c_uint16), ("shard_index", C.c_uint16), ("symbol_size", C.c_uint32),
                ("original_length", C.c_uint64)]


def load():
    """Load the in-tree shared object (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1709_00178_b200.build` "
                          "(there is no CPU fallback for the codec)")
    lib = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    P = C.POINTER
    lib.pyrit_version.restype = C.c_char_p
    lib.pyrit_strerror.restype = C.c_char_p
    lib.pyrit_strerror.argtypes = [i32]
    lib.pyrit_plan_create.argtypes = [P(pyrit_field), u32, vp, u32, u32, u32, u32, P(vp)]
    lib.pyrit_plan_encode.argtypes = [P(pyrit_code), P(vp)]
    lib.pyrit_plan_decode.argtypes = [P(pyrit_code), vp, u32, P(vp), vp, vp]
    lib.pyrit_plan_get_stats.argtypes = [vp, P(pyrit_plan_stats)]
    lib.pyrit_plan_reps.argtypes = [vp, vp]
    lib.pyrit_plan_key.argtypes = [vp, vp, C.c_size_t]
    lib.pyrit_plan_inject_fault.argtypes = [vp, u32, u32]
    lib.pyrit_plan_source.argtypes = [vp, u32, vp, C.c_size_t, P(C.c_size_t), vp, C.c_size_t]
    lib.pyrit_plan_interpret.argtypes = [vp, vp, vp, u64, u64, u64]
    lib.pyrit_plan_destroy.argtypes = [vp]
    lib.pyrit_plan_destroy.restype = None
    lib.pyrit_cu_apply.argtypes = [vp, vp, vp, u64, u64, u64, vp]
    lib.pyrit_cu_prepare.argtypes = [vp]
    lib.pyrit_cu_encode.argtypes = [P(pyrit_code), vp, vp, u64, vp]
    lib.pyrit_cu_encode_crs.argtypes = [P(pyrit_code), vp, vp, u64, vp]
    lib.pyrit_encode_crs_host.argtypes = [P(pyrit_code), vp, vp, u64, i32]
    lib.pyrit_encode_host_devices.argtypes = [P(pyrit_code), vp, vp, u64, vp, u32]
    lib.pyrit_decode_host_devices.argtypes = [P(pyrit_code), vp, vp, u32, u64, vp, u32]
    lib.pyrit_cu_decode.argtypes = [P(pyrit_code), vp, vp, u32, u64, vp]
    lib.pyrit_encode_host.argtypes = [P(pyrit_code), vp, vp, u64, i32]
    lib.pyrit_decode_host.argtypes = [P(pyrit_code), vp, vp, u32, u64, i32]
    lib.pyrit_set_host_chunk.argtypes = [u64]
    lib.pyrit_cu_fill.argtypes = [u64, u64, vp, u64, u64, u64, vp]
    lib.pyrit_cu_digest.argtypes = [vp, u64, u64, vp, vp]
    lib.pyrit_set_lanes.argtypes = [u32]
    lib.pyrit_set_kernel_dir.argtypes = [C.c_char_p]
    lib.pyrit_set_kernel_mode.argtypes = [i32]
    lib.pyrit_cu_last_launch.argtypes = [vp, C.c_size_t, vp, vp]
    lib.pyrit_jit_compiles.restype = u64
    lib.pyrit_jit_time.argtypes = [P(C.c_double), P(C.c_double)]
    lib.pyrit_rt_interpret.argtypes = [vp, vp, vp, u64, u64, u64, u64, u64, u64]
    lib.pyrit_rt_plan_info.argtypes = [vp, P(u32)]
    lib.pyrit_plan_from_ringmat.argtypes = [P(pyrit_ringmat), vp]
    lib.pyrit_warmup.argtypes = [i32]
    lib.pyrit_numa_bind_thread.argtypes = [i32]
    lib.pyrit_bind_thread_cpulist.argtypes = [C.c_char_p]
    lib.pyrit_cu_apply_ringmat.argtypes = [P(pyrit_ringmat), vp, vp, u64, u64, u64, vp]
    lib.pyrit_kernel_launches.restype = u64
    lib.pyrit_field_named.argtypes = [C.c_char_p, P(pyrit_field)]
    lib.pyrit_field_validate.argtypes = [P(pyrit_field)]
    lib.pyrit_gf_mul.argtypes = [P(pyrit_field), u32, u32, P(u32)]
    lib.pyrit_gf_inv.argtypes = [P(pyrit_field), u32, P(u32)]
    lib.pyrit_sparse_transform.argtypes = [P(pyrit_field), u32, P(u32)]
    lib.pyrit_fold_table.argtypes = [P(pyrit_field), vp]
    lib.pyrit_cauchy_parity_matrix.argtypes = [P(pyrit_code), vp]
    lib.pyrit_decode_matrix.argtypes = [P(pyrit_code), vp, vp, P(u32)]
    lib.pyrit_repair_matrix.argtypes = [P(pyrit_code), vp, u32, vp, vp, vp]
    lib.pyrit_cu_apply_batch.argtypes = [vp, vp, vp, u64, u64, u64, u64, u64, u64, vp]
    lib.pyrit_cu_encode_batch.argtypes = [P(pyrit_code), vp, vp, u64, u64, u64, u64, vp]
    lib.pyrit_cu_decode_batch.argtypes = [P(pyrit_code), vp, vp, u32, u64, u64, u64, vp]
    lib.pyrit_crc32.argtypes = [vp, C.c_size_t]
    lib.pyrit_crc32.restype = u32
    lib.pyrit_header_serialize.argtypes = [P(pyrit_shard_header), vp]
    lib.pyrit_header_parse.argtypes = [vp, C.c_size_t, P(pyrit_shard_header)]
    lib.pyrit_field_id.argtypes = [P(pyrit_field), P(C.c_uint8)]
    lib.pyrit_field_from_id.argtypes = [C.c_uint8, P(pyrit_field)]
    lib.pyrit_shard_path.argtypes = [C.c_char_p, C.c_char_p, u32, vp, C.c_size_t]
    lib.pyrit_encode_file.argtypes = [P(pyrit_code), C.c_char_p, C.c_char_p, u32, i32]
    lib.pyrit_decode_file.argtypes = [P(C.c_char_p), u32, C.c_char_p, i32]
    lib.pyrit_set_file_chunk.argtypes = [u64]
    lib.pyrit_plan_from_schedule.argtypes = [P(pyrit_field), u32, u32, vp, C.c_size_t, vp, P(vp)]
    lib.pyrit_apply_host.argtypes = [vp, vp, vp, u64, u64, u64, i32]
    lib.pyrit_jit_info.argtypes = [vp, C.c_size_t]
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().pyrit_strerror(rc).decode(errors="replace")
        raise PyritError(rc, msg)

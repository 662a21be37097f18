"""The C-ABI library on a machine without a GPU: it loads, exports every entry
point include/pyrit_b200.h declares, and its host-only entry points behave
(error codes mirror Errc, errors.hpp:12-24).  No device calls here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1709_00178_b200 as P
from paper_1709_00178_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pyrit_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pyrit_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pyrit_cu_apply", "pyrit_cu_encode", "pyrit_cu_decode", "pyrit_encode_host", "pyrit_decode_host",
                 "pyrit_plan_create", "pyrit_cauchy_parity_matrix", "pyrit_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(pyrit_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and nothing else leaks (internals are hidden; static cudart is excluded)
    assert all(n.startswith("pyrit_") for n in re.findall(r"\sT\s(\S+)", out))
    lib = L.load()
    for n in declared_functions():
        assert hasattr(lib, n)
    assert set(L.EXPORTS) <= set(declared_functions())


def test_version_and_strerror():
    lib = L.load()
    assert b"sm_100a" in lib.pyrit_version()
    assert lib.pyrit_strerror(0) == b"ok"
    assert lib.pyrit_strerror(3).startswith(b"TooManySymbols")
    assert lib.pyrit_strerror(6).startswith(b"InsufficientShards")


def test_return_codes_are_errc_plus_one():
    lib = L.load()
    code = L.pyrit_code(13, 4, L.pyrit_field(4, 5, 0, 1, 4, 0x1F), 0)
    out = np.zeros(64, np.uint16)
    assert lib.pyrit_cauchy_parity_matrix(C.byref(code), out.ctypes.data) == 3  # TooManySymbols
    code = L.pyrit_code(0, 4, L.pyrit_field(4, 5, 0, 1, 4, 0x1F), 0)
    assert lib.pyrit_cauchy_parity_matrix(C.byref(code), out.ctypes.data) == 11  # InvalidArgument
    bad = L.pyrit_field(4, 6, 0, 1, 4, 0x1F)  # p does not divide x^6 + 1
    assert lib.pyrit_field_validate(C.byref(bad)) == 11
    f = L.pyrit_field()
    assert lib.pyrit_field_named(b"gf256_r17", C.byref(f)) == 0 and (f.w, f.n, f.modulus) == (8, 17, 0x139)
    assert lib.pyrit_field_named(b"nope", C.byref(f)) == 11
    # symbol size rules of SymbolBuffer (codec.hpp:28-30) are checked before any device work
    code = L.pyrit_code(4, 2, L.pyrit_field(4, 5, 0, 1, 4, 0x1F), 0)
    ptrs = (C.c_void_p * 6)()
    assert lib.pyrit_cu_encode(C.byref(code), ptrs, ptrs, 12, None) == 4  # BufferShape (12 % 8)
    assert lib.pyrit_cu_encode(C.byref(code), ptrs, ptrs, 0, None) == 4
    er = (C.c_uint32 * 3)(0, 1, 2)
    assert lib.pyrit_cu_decode(C.byref(code), ptrs, er, 3, 16, None) == 6  # InsufficientShards


def test_plans_describe_themselves():
    plan = P.Plan.encode(P.CodeSpec(16, 4, P.FieldSpec.aop(12)))
    st = plan.stats()
    assert (st["rows"], st["cols"], st["ref_region_ops"]) == (4, 16, 2808)
    name, src = plan.source(L.SOURCE_STAGED)
    assert name.startswith("pyrit_ring_k16_e4_w12_n13_tmt") and "cp.async.bulk.tensor.3d" in src
    name8, src8 = plan.source(L.SOURCE_STAGED + 8)  # 8-byte aligned strips: cp.async producer
    assert "_cpa8_" in name8 and "cp.async.ca.shared.global" in src8
    assert "mbarrier.try_wait.parity" in src and "__grid_constant__" in src
    name1, src1 = plan.source(1)
    assert "_L1_" in name1 and "ld.global.nc" in src1
    assert plan.key().startswith("w12n13_4x16_")
    assert plan.reps().shape == (4, 16)


def test_tuned_table_entries_match_current_plan_keys():
    from paper_1709_00178_b200.workloads import WORKLOADS
    keys = set()
    for line in open(os.path.join(ROOT, "paper_1709_00178_b200", "tuned.tsv")):
        if line.strip() and not line.startswith("#"):
            keys.add(line.split()[0])
    current = set()
    for cfg in (1, 2, 3, 4, 5):
        wl = WORKLOADS[cfg]
        plan = P.Plan.encode(wl.code) if wl.op == "encode" else P.Plan.decode(wl.code, wl.erased)
        current.add(plan.key())
    # the paper's large GF(2^6) codes (Fig. 2/3): (60,40) embedding and (60,20) parity
    for k, r, t in ((40, 20, 0), (20, 40, 1)):
        current.add(P.Plan.encode(P.CodeSpec(k, r, P.FieldSpec.gf64_esp(), P.TransformKind(t))).key())
    assert keys <= current, keys - current  # no stale rows (representatives changed)


def test_null_arguments_are_errors_not_crashes():
    """Every host entry point reports InvalidArgument (1 + Errc) for null outputs."""
    lib = L.load()
    f = P.FieldSpec.gf16_aop().c()
    code = P.CodeSpec(4, 2, P.FieldSpec.gf16_aop()).c()
    inv = 11  # 1 + Errc::InvalidArgument
    assert lib.pyrit_gf_mul(C.byref(f), 2, 3, None) == inv
    assert lib.pyrit_gf_inv(C.byref(f), 2, None) == inv
    assert lib.pyrit_sparse_transform(C.byref(f), 2, None) == inv
    assert lib.pyrit_fold_table(C.byref(f), None) == inv
    assert lib.pyrit_cauchy_parity_matrix(C.byref(code), None) == inv
    assert lib.pyrit_decode_matrix(C.byref(code), None, None, None) == inv
    assert lib.pyrit_repair_matrix(C.byref(code), None, 1, None, None, None) == inv
    assert lib.pyrit_header_parse(None, 29, None) == inv
    assert lib.pyrit_encode_file(None, b"x", b"y", 16, 0) == inv
    assert lib.pyrit_decode_file(None, 1, b"out", 0) == inv
    assert lib.pyrit_cu_apply(None, None, None, 16, 0, 16, None) == inv
    assert lib.pyrit_cu_apply_batch(None, None, None, 16, 0, 16, 1, 0, 0, None) == inv


def test_jit_uses_the_toolkit_nvrtc_even_after_another_was_loaded():
    """A torch process may already hold its own (older) libnvrtc.so.12; kernels that are not prebuilt
    must still be compiled by the toolkit NVRTC the prebuilt ones came from (profiles/r01_s3/jit/)."""
    import glob
    import subprocess
    import sys
    others = [p for p in glob.glob(os.path.join(os.path.dirname(np.__file__), "..", "nvidia", "cuda_nvrtc", "lib",
                                                "libnvrtc.so.12"))]
    pre = f"import ctypes; ctypes.CDLL({others[0]!r}, mode=ctypes.RTLD_GLOBAL); " if others else ""
    code = pre + "import paper_1709_00178_b200 as P; print(P.jit_info())"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, check=True).stdout
    assert out.startswith("nvrtc 12.") and "/usr/local/cuda" in out, out


def test_header_is_plain_c(tmp_path):
    """include/pyrit_b200.h compiles as C11 with warnings as errors, and a C program links and runs
    against the library (host-side entry points only)."""
    exe = tmp_path / "c_header_check"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_header_check.c"), "-o", str(exe),
                    "-L", os.path.dirname(L.LIB_PATH), "-lpyrit_b200", f"-Wl,-rpath,{os.path.dirname(L.LIB_PATH)}"],
                   check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stderr)
    assert "sm_100a" in out.stdout


def test_numa_bind_without_a_device_changes_nothing():
    """pyrit_numa_bind_thread is best effort: with no usable device (or an unknown node) it
    returns -1 and leaves the calling thread's affinity as it was."""
    lib = L.load()
    before = os.sched_getaffinity(0)
    node = lib.pyrit_numa_bind_thread(1 << 20)
    assert node == -1
    assert os.sched_getaffinity(0) == before


def test_bind_thread_cpulist():
    """The affinity step of pyrit_numa_bind_thread on its own: a sysfs-style CPU list is
    intersected with the thread's cpuset; a disjoint, empty or malformed list changes nothing."""
    import threading
    lib = L.load()
    allowed = sorted(os.sched_getaffinity(0))
    seen = {}

    def worker():  # affinity is per thread: do it off the main thread
        lo = allowed[0]
        seen["one"] = (lib.pyrit_bind_thread_cpulist(f"{lo}\n".encode()), os.sched_getaffinity(0))
        seen["disjoint"] = (lib.pyrit_bind_thread_cpulist(b"100000-100003"), os.sched_getaffinity(0))
        seen["empty"] = lib.pyrit_bind_thread_cpulist(b"")
        seen["junk"] = lib.pyrit_bind_thread_cpulist(b"abc")

    t = threading.Thread(target=worker)
    t.start()
    t.join()
    assert seen["one"] == (1, {allowed[0]})
    assert seen["disjoint"] == (-1, {allowed[0]})
    assert seen["empty"] == -1 and seen["junk"] == -1
    assert sorted(os.sched_getaffinity(0)) == allowed  # the main thread is untouched

    def ranges():
        seen["range"] = (lib.pyrit_bind_thread_cpulist(f"{allowed[0]}-{allowed[-1]},{allowed[0]}".encode()),
                         os.sched_getaffinity(0))

    t = threading.Thread(target=ranges)
    t.start()
    t.join()
    assert seen["range"][1] == set(allowed)

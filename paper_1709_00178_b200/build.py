"""Build libpyrit_b200.so in-tree (sm_100a) and prebuild the generated ring kernels.

    python -m paper_1709_00178_b200.build [--force] [--no-prebuild]

Steps
  1. g++ (C++20) compiles the host algebra, program compiler, runtime, pipeline
     and C ABI; nvcc compiles the ahead-of-time kernels (kernels.cu) with
     -gencode arch=compute_100a,code=sm_100a -lineinfo; both link into
     paper_1709_00178_b200/libpyrit_b200.so (static cudart, NVRTC, hidden internals).
  2. For the BASELINE.json encode/decode programs, the library's own code
     generator emits CUDA C which nvcc compiles to
     paper_1709_00178_b200/kernels/<kernel>.cubin; the runtime loads those before
     falling back to NVRTC, so no JIT happens for the benchmarked plans.
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libpyrit_b200.so")
HELPER = os.path.join(os.path.dirname(LIB), "pyrit_jit_helper")
KDIR = os.path.join(PKG, "kernels")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SOURCES = ["algebra.cpp", "program.cpp", "runtime.cpp", "pipeline.cpp", "plans.cpp", "container.cpp", "hostpool.cpp", "capi.cpp"]
# paired-shift cases of the runtime-matrix kernel: shifts up to this far apart share one
# case (kernels.hpp PYRIT_RT_PAIR_D); a build-time constant of the library
# (default: the #define in csrc/kernels.hpp; PYRIT_B200_BUILD_RT_PAIR_D overrides it for A/B builds)
def _default_pair_d() -> int:
    import re

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "kernels.hpp")) as f:
        return int(re.search(r"#define PYRIT_RT_PAIR_D (\d+)", f.read()).group(1))


RT_PAIR_D = int(os.environ.get("PYRIT_B200_BUILD_RT_PAIR_D", "") or _default_pair_d())
RT_PAIR_AOP_ALL = int(os.environ.get("PYRIT_B200_BUILD_RT_PAIR_AOP_ALL", "0"))
CUDA_SOURCES = ["kernels.cu", "ring_rt.cu", "ring_rt_w4_n5.cu", "ring_rt_w6_n9.cu", "ring_rt_w8_n17.cu",
                "ring_rt_w10_n11.cu", "ring_rt_w12_n13.cu"]
HEADERS = ["algebra.hpp", "program.hpp", "runtime.hpp", "pipeline.hpp", "plans.hpp", "container.hpp", "kernels.hpp",
           "ring_rt.cuh"]


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force=False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "pyrit_b200.h")]
    stamp = os.path.join(BUILD, "rt_pair_d.stamp")  # objects depend on the -D value they were built with
    if not os.path.exists(stamp) or open(stamp).read() != f"{RT_PAIR_D},{RT_PAIR_AOP_ALL}":
        with open(stamp, "w") as f:
            f.write(f"{RT_PAIR_D},{RT_PAIR_AOP_ALL}")
    hdrs.append(stamp)
    objs = []
    for src in HOST_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run(["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
                  f"-I{CUDA}/include", f"-DPYRIT_RT_PAIR_D={RT_PAIR_D}", f"-DPYRIT_RT_PAIR_AOP_ALL={RT_PAIR_AOP_ALL}", f'-DPYRIT_NVRTC_PATH="{CUDA}/lib64/libnvrtc.so.12"', "-c", s, "-o", o])
        objs.append(o)
    # dispatch tables of the runtime-matrix ring kernel (generated, build/generated)
    gen_dir = os.path.join(BUILD, "generated")
    os.makedirs(gen_dir, exist_ok=True)
    inc = os.path.join(gen_dir, "ring_rt_ops.inc")
    gen = os.path.join(PKG, "gen_ring_rt.py")
    sys.path.insert(0, ROOT)
    from paper_1709_00178_b200 import gen_ring_rt

    text = gen_ring_rt.generate(RT_PAIR_D, bool(RT_PAIR_AOP_ALL))
    if force or not os.path.exists(inc) or open(inc).read() != text:
        with open(inc, "w") as f:
            f.write(text)
    # the CUDA translation units (one per runtime-matrix ring geometry) compile in parallel
    jobs = []
    for src in CUDA_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s, inc] + hdrs):
            jobs.append([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", f"-I{gen_dir}", f"-DPYRIT_RT_PAIR_D={RT_PAIR_D}", f"-DPYRIT_RT_PAIR_AOP_ALL={RT_PAIR_AOP_ALL}",
                         "-Xcompiler",
                         "-fPIC,-fvisibility=hidden", "-c", s, "-o", o])
        objs.append(o)
    if jobs:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            for f in [ex.submit(_run, j) for j in jobs]:
                f.result()
    # the background-compile helper (tiered compilation runs NVRTC in its own process)
    helper_src = os.path.join(CSRC, "jit_helper.cpp")
    if force or _stale(HELPER, [helper_src]):
        _run(["g++", "-std=c++20", "-O2", f"-I{CUDA}/include", f'-DPYRIT_NVRTC_PATH="{CUDA}/lib64/libnvrtc.so.12"',
              helper_src, "-o", HELPER, "-ldl"])
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static", f"-L{CUDA}/lib64",
              "-Xlinker", "--exclude-libs,ALL", "-ldl", "-lpthread", "-lrt"])
    return LIB


# (name, field, k, r, erased) -- the programs bench.py and the GPU tests run
def baseline_programs():
    gf16 = (4, 5, 0, 1, 4, 0x1F)
    gf256 = (8, 17, 0, 1, 8, 0x139)
    gf1024 = (10, 11, 0, 1, 10, 0x7FF)
    gf4096 = (12, 13, 0, 1, 12, 0x1FFF)
    return [
        ("cfg1", gf16, 4, 2, None),
        ("cfg2", gf256, 10, 4, None),
        ("cfg3", gf1024, 12, 4, None),
        ("cfg4-dec", gf256, 10, 4, (1, 6, 9, 10)),
        ("cfg4-dec-data", gf256, 10, 4, (0, 1, 2, 3)),
        ("cfg5", gf4096, 16, 4, None),
    ]


def prebuild_kernels(lanes=(100, 1), force=False) -> list[str]:
    """Generate + nvcc-compile the BASELINE plans' kernels into kernels/*.cubin."""
    sys.path.insert(0, ROOT)
    from paper_1709_00178_b200 import _lib as L  # noqa: E402

    lib = L.load()
    os.makedirs(KDIR, exist_ok=True)
    src_dir = os.path.join(BUILD, "generated")
    os.makedirs(src_dir, exist_ok=True)
    built = []
    keys = []
    for tag, fld, k, r, erased in baseline_programs():
        code = L.pyrit_code(k, r, L.pyrit_field(*fld), 0)
        plan = C.c_void_p()
        if erased is None:
            L.check(lib.pyrit_plan_encode(C.byref(code), C.byref(plan)))
        else:
            er = (C.c_uint32 * len(erased))(*erased)
            L.check(lib.pyrit_plan_decode(C.byref(code), er, len(erased), C.byref(plan), None, None))
        try:
            kb = C.create_string_buffer(128)
            L.check(lib.pyrit_plan_key(plan, kb, 128))
            keys.append(kb.value.decode())
            for ln in lanes:
                size = C.c_size_t(0)
                name = C.create_string_buffer(128)
                rc = lib.pyrit_plan_source(plan, ln, None, 0, C.byref(size), name, 128)
                if rc == 4 and ln in (L.SOURCE_STAGED, L.SOURCE_STAGED + 1):
                    continue  # tiles do not fit in shared memory: direct kernel only
                L.check(rc)
                buf = C.create_string_buffer(size.value + 1)
                L.check(lib.pyrit_plan_source(plan, ln, buf, size.value + 1, None, None, 0))
                nm = name.value.decode()
                cu = os.path.join(src_dir, nm + ".cu")
                cubin = os.path.join(KDIR, nm + ".cubin")
                with open(cu, "w") as f:
                    f.write(buf.value.decode())
                if force or not os.path.exists(cubin):
                    _run([NVCC, "-cubin", *ARCH, "-lineinfo", "-O3", "-diag-suppress", "177", "-Xptxas", "-v", cu,
                          "-o", cubin])
                built.append(cubin)
        finally:
            lib.pyrit_plan_destroy(plan)
    # plan keys with prebuilt kernels: decode patterns listed here run their
    # specialised kernel, every other pattern the runtime-matrix kernel
    with open(os.path.join(KDIR, "prebuilt.tsv"), "w") as f:
        f.write("\n".join(keys) + "\n")
    # cubins of older generator versions are never loaded again: drop them
    for f in os.listdir(KDIR):
        if f.endswith(".cubin") and os.path.join(KDIR, f) not in built:
            os.remove(os.path.join(KDIR, f))
    return built


def build_test_tools(force=False) -> str:
    """tests/sanitize_check.cpp -> build/sanitize_check (compute-sanitizer driver, test infrastructure)."""
    src = os.path.join(ROOT, "tests", "sanitize_check.cpp")
    out = os.path.join(BUILD, "sanitize_check")
    if force or _stale(out, [src, LIB, os.path.join(ROOT, "include", "pyrit_b200.h")]):
        _run([NVCC, *ARCH, "-O2", "-std=c++17", f"-I{os.path.join(ROOT, 'include')}", src, "-o", out, f"-L{PKG}",
              "-lpyrit_b200", "-Xlinker", "-rpath,$ORIGIN/../paper_1709_00178_b200"])
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--no-prebuild", action="store_true")
    ap.add_argument("--lanes", default="100,1",
                    help="100 = staged kernel, 101 = staged for equally spaced inputs, 1/2/4 = direct")
    a = ap.parse_args(argv)
    build_library(a.force)
    build_test_tools(a.force)
    if not a.no_prebuild:
        prebuild_kernels(tuple(int(x) for x in a.lanes.split(",")), a.force)


if __name__ == "__main__":
    main()

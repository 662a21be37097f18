"""Host sanitizers: the library's host sources under
-fsanitize=address,undefined and under -fsanitize=thread.

tests/host_sanitize_check.cpp walks every C-ABI entry point that needs no
device (field algebra, matrices, plan compilation, both host interpreters,
CUDA source generation, fault injection, shard headers with a byte fuzz,
argument errors) and a multi-threaded section over the lazily built tables
and the plan cache.  Each sanitizer build compiles csrc/*.cpp afresh (the
CUDA objects come from the normal build) and must run to "0 failed" with no
sanitizer report.  compute-sanitizer is refused by the GPU pool
(profiles/r02/sanitize/), so this is the memory-safety check of the host side
and tests/sanitize_check.cpp (allocation-exact buffers) that of the kernels.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1709_00178_b200", "csrc")
BUILD = os.path.join(ROOT, "build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")

HOST = ["algebra", "program", "runtime", "pipeline", "plans", "container", "hostpool", "capi"]
CUDA_OBJS = ["kernels.cu.o", "ring_rt.cu.o", "ring_rt_w4_n5.cu.o", "ring_rt_w6_n9.cu.o", "ring_rt_w8_n17.cu.o",
             "ring_rt_w10_n11.cu.o", "ring_rt_w12_n13.cu.o"]
MODES = {
    "asan": ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined"],
    "tsan": ["-fsanitize=thread"],
}


def _build(mode: str, driver: str = "host_sanitize_check") -> str:
    out = os.path.join(BUILD, mode)
    os.makedirs(out, exist_ok=True)
    flags = ["-std=c++20", "-O1", "-g", "-fno-omit-frame-pointer", *MODES[mode]]

    def cc(name):
        obj = os.path.join(out, name + ".o")
        subprocess.run(["g++", *flags, f"-I{CUDA}/include", f'-DPYRIT_NVRTC_PATH="{CUDA}/lib64/libnvrtc.so.12"', "-c",
                        os.path.join(CSRC, name + ".cpp"), "-o", obj], check=True, capture_output=True, text=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(HOST), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(cc, HOST))
    exe = os.path.join(out, driver)
    subprocess.run(["g++", *flags, f"-I{os.path.join(ROOT, 'include')}", f"-I{CUDA}/include",
                    os.path.join(ROOT, "tests", driver + ".cpp"),
                    *objs, *[os.path.join(BUILD, o) for o in CUDA_OBJS], f"-L{CUDA}/lib64", "-lcudart_static", "-ldl",
                    "-lpthread", "-lrt", "-o", exe], check=True, capture_output=True, text=True)
    return exe


@pytest.fixture(scope="module")
def cuda_objects():
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    missing = [o for o in CUDA_OBJS if not os.path.exists(os.path.join(BUILD, o))]
    if missing:  # the normal build leaves them in build/
        from paper_1709_00178_b200 import build as B

        B.build_library()
    return True


@pytest.mark.parametrize("mode", sorted(MODES))
def test_host_sources_clean_under_sanitizer(cuda_objects, mode):
    try:
        exe = _build(mode)
    except subprocess.CalledProcessError as e:  # a toolchain without the sanitizer runtime
        if "cannot find -lasan" in e.stderr or "cannot find -ltsan" in e.stderr or "cannot find -lubsan" in e.stderr:
            pytest.skip("sanitizer runtime not installed")
        raise AssertionError(e.stderr[-4000:])
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:halt_on_error=1", UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1",
               TSAN_OPTIONS="halt_on_error=1:second_deadlock_stack=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " 0 failed" in r.stdout, tail
    for word in ("ERROR: AddressSanitizer", "runtime error:", "WARNING: ThreadSanitizer", "ERROR: LeakSanitizer"):
        assert word not in r.stderr, tail


@pytest.mark.gpu
def test_host_buffer_paths_clean_under_asan_on_gpu(cuda_objects):
    """tests/host_sanitize_gpu.cpp: the host-buffer C ABI (pipeline, shards over devices, stripe
    batches, runtime-matrix decode, file codec, concurrent callers) with the host sources under
    ASan+UBSan, on the device, every result checked against the host interpreter."""
    exe = _build("asan", "host_sanitize_gpu")
    env = dict(os.environ, ASAN_OPTIONS="protect_shadow_gap=0:detect_leaks=0:halt_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", PYRIT_B200_JIT_CACHE="0")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " 0 failed" in r.stdout, tail
    for word in ("ERROR: AddressSanitizer", "runtime error:"):
        assert word not in r.stderr, tail

"""GPU parity of the runtime-matrix ring kernel (csrc/ring_rt.cu, kernel mode 4).

One ahead-of-time kernel per ring geometry applies any matrix passed in its
kernel parameters; these tests hold it bit-exact against the oracle
(oracle/, pinned to the reference in test_oracle.py) over the BASELINE fields,
both transforms, every output count up to and past one launch's accumulators,
k up to 64, stripe batches, column windows, in-place repair, and every erasure
pattern of the (10, 4) GF(2^8)/R_{2,17} code with zero NVRTC compiles.
"""
from __future__ import annotations

import itertools
import os
import random

import numpy as np
import pytest

import paper_1709_00178_b200 as P
from paper_1709_00178_b200 import _lib as L
from paper_1709_00178_b200.workloads import WORKLOADS
from tests.helpers import G16, G64, G256, G1024, G4096, oracle_encode, oracle_ring, rand_symbols, seeded_symbols

pytestmark = pytest.mark.gpu

FIELDS = [G16, G64, G256, G1024, G4096]


class mode:
    def __init__(self, m):
        self.m = m

    def __enter__(self):
        L.check(L.load().pyrit_set_kernel_mode(self.m))

    def __exit__(self, *exc):
        L.check(L.load().pyrit_set_kernel_mode(0))


def run_plan(cuda, plan, src: np.ndarray, rows: int, strip: int, off: int = 0, length: int | None = None,
             init: np.ndarray | None = None) -> np.ndarray:
    import torch
    d = torch.from_numpy(np.ascontiguousarray(src)).to(cuda)
    out = (torch.from_numpy(init).to(cuda) if init is not None
           else torch.zeros((rows, src.shape[1]), dtype=torch.uint8, device=cuda))
    plan.apply([d[j].data_ptr() for j in range(d.shape[0])], [out[i].data_ptr() for i in range(rows)], strip, off,
               length)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def rt_launched() -> str:
    k = P.Plan.last_launch()["kernel"]
    assert k.startswith("pyrit_ring_rt_"), k
    return k


@pytest.mark.parametrize("f", FIELDS, ids=lambda f: f"w{f.w}n{f.n}")
@pytest.mark.parametrize("kind", [0, 1])
def test_random_matrices_match_oracle(cuda, f, kind):
    """Random GF(2^w) matrices, e = 1 .. past one launch's outputs (output groups of one launch,
    then further launches), k up to 64."""
    rng = np.random.default_rng(1000 * f.w + kind)
    for e, k in [(1, 1), (2, 3), (3, 7), (4, 10), (5, 16), (8, 12), (9, 5), (17, 3), (4, 64), (2, 33), (20, 40),
                 (40, 3)]:
        m = rng.integers(0, 1 << f.w, (e, k), dtype=np.uint16)
        m[rng.random((e, k)) < 0.1] = 0  # zero entries: no ops
        plan = P.Plan.create(f, m, P.TransformKind(kind))
        ss = f.w * 16 * 80 * 3  # 3 full 2 KiB tiles + part of a fourth per strip (V=2)
        data = rand_symbols(k, ss, int(rng.integers(1 << 30)))
        with mode(4):
            got = run_plan(cuda, plan, data, e, ss // f.w)
            rt_launched()
        np.testing.assert_array_equal(got, oracle_ring(f, m, data, kind=kind), err_msg=f"e={e} k={k}")


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_baseline_encode_small(cuda, cfg):
    wl = WORKLOADS[cfg]
    ss = wl.fld.w * 4096 * 3
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    C = P.cauchy_parity_matrix(wl.code)
    plan = P.Plan.encode(wl.code)
    with mode(4):
        got = run_plan(cuda, plan, data, wl.m, ss // wl.fld.w)
        rt_launched()
    np.testing.assert_array_equal(got, oracle_ring(wl.fld, C, data))
    # and the field-level oracle (codec.hpp:444-469) on the same bytes
    np.testing.assert_array_equal(got, oracle_encode(wl.fld, C, data))


@pytest.mark.parametrize("f", [G16, G256, G4096], ids=lambda f: f"w{f.w}n{f.n}")
def test_windows_and_batches(cuda, f):
    """Column windows [off, off+len) and stripe batches with pitches (one launch)."""
    import torch
    rng = np.random.default_rng(f.w)
    k, e = 6, 3
    m = rng.integers(1, 1 << f.w, (e, k), dtype=np.uint16)
    plan = P.Plan.create(f, m)
    strip = 16 * 700
    ss = f.w * strip
    data = rand_symbols(k, ss, 3)
    init = rand_symbols(e, ss, 4)  # bytes outside the window stay as they were
    want = oracle_ring(f, m, data)
    with mode(4):
        for off, length in [(0, 16), (16 * 37, 16 * 300), (strip - 16 * 129, 16 * 129), (0, strip)]:
            got = run_plan(cuda, plan, data, e, strip, off, length, init=init)
            rt_launched()
            exp = init.copy()
            for i in range(e):
                for s in range(f.w):
                    a = s * strip + off
                    exp[i, a:a + length] = want[i, a:a + length]
            np.testing.assert_array_equal(got, exp, err_msg=f"off={off} len={length}")
        # stripe batch: nb stripes of k symbols each, in pitch = k*ss + 64, out pitch = e*ss + 32
        nb = 5
        ipitch, opitch = k * ss + 64, e * ss + 32
        src = rand_symbols(1, nb * ipitch, 9)[0]
        d = torch.from_numpy(src).to(cuda)
        out = torch.zeros(nb * opitch, dtype=torch.uint8, device=cuda)
        plan.apply_batch([d.data_ptr() + j * ss for j in range(k)], [out.data_ptr() + i * ss for i in range(e)],
                         strip, nb, ipitch, opitch)
        torch.cuda.synchronize()
        rt_launched()
        got = out.cpu().numpy()
    for b in range(nb):
        syms = np.stack([src[b * ipitch + j * ss: b * ipitch + (j + 1) * ss] for j in range(k)])
        exp = oracle_ring(f, m, syms)
        for i in range(e):
            np.testing.assert_array_equal(got[b * opitch + i * ss: b * opitch + (i + 1) * ss], exp[i])


def test_all_erasure_patterns_config4_no_compile(cuda):
    """Every erasure pattern (weight 1..4, 1470 of them) of the (10, 4) GF(2^8)/R_{2,17} code repairs
    bit-exact through decode() in the default mode -- ad-hoc patterns run on the runtime kernel -- and
    the whole sweep compiles nothing (pyrit_jit_compiles unchanged)."""
    import torch
    wl = WORKLOADS[4]
    ss = wl.fld.w * 16 * 96
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    full = np.concatenate([data, oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data)])
    ref = torch.from_numpy(full).to(cuda)
    work = ref.clone()
    lib = L.load()
    jit0 = lib.pyrit_jit_compiles()
    kdir = os.path.join(os.path.dirname(P.__file__), "kernels")
    n = 0
    for wgt in range(1, 5):
        for er in itertools.combinations(range(14), wgt):
            work[list(er)] = 0xA5
            P.decode(work, er, wl.code)
            # a pattern whose program has a prebuilt kernel (the benchmarked ones, or all
            # parity erased = the encode program) runs it; every other one the runtime kernel
            k = P.Plan.last_launch()["kernel"]
            if not os.path.exists(os.path.join(kdir, k + ".cubin")):
                rt_launched()
            n += 1
            if n % 64 == 0 or wgt < 4:
                torch.cuda.synchronize()
                assert torch.equal(work, ref), er
    torch.cuda.synchronize()
    assert torch.equal(work, ref)
    assert n == 1470
    assert lib.pyrit_jit_compiles() == jit0, "a decode pattern was compiled"


def test_in_place_repair_aliasing(cuda):
    """decode() passes one buffer as input and output: exact column-for-column aliasing is allowed."""
    wl = WORKLOADS[4]
    ss = wl.fld.w * 16 * 200
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    full = np.concatenate([data, oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data)])
    import torch
    for er in [(2, 5, 11, 13), (0, 9), (12,)]:
        w = torch.from_numpy(full.copy()).to(cuda)
        w[list(er)] = 0
        with mode(4):
            P.decode(w, er, wl.code)
            rt_launched()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(w.cpu().numpy(), full)


def test_misaligned_falls_back(cuda):
    """Launches the runtime kernel cannot take (8-byte aligned strips) still run exactly."""
    f = G256
    m = np.array([[3, 7, 11], [200, 1, 9]], dtype=np.uint16)
    plan = P.Plan.create(f, m)
    ss = f.w * 8 * 301
    data = rand_symbols(3, ss, 12)
    with mode(4):
        got = run_plan(cuda, plan, data, 2, ss // f.w)
        assert not P.Plan.last_launch()["kernel"].startswith("pyrit_ring_rt_")
    np.testing.assert_array_equal(got, oracle_ring(f, m, data))


def test_full_size_config4_random_patterns(cuda):
    """Config 4 at its full 64 MiB fragments: random data+parity patterns on the runtime kernel
    agree with the specialised prebuilt kernel's pattern and with the original symbols."""
    import torch
    wl = WORKLOADS[4]
    buf = torch.empty((14, wl.frag), dtype=torch.uint8, device=cuda)
    for j in range(wl.k):
        P.fill(buf[j], wl.seed, j, valid=wl.valid)
    P.encode(buf[: wl.k], wl.code)  # warm
    buf[wl.k:] = P.encode(buf[: wl.k], wl.code)
    ref = buf.clone()
    rng = random.Random(3)
    for er in [(0, 1, 2, 3)] + [tuple(sorted(rng.sample(range(14), 4))) for _ in range(3)]:
        buf[list(er)] = 0
        with mode(4):
            P.decode(buf, er, wl.code)
            rt_launched()
        torch.cuda.synchronize()
        assert torch.equal(buf, ref), er


def test_hot_pattern_gets_specialised_kernel(cuda, tmp_path):
    """With tiered compilation on, a decode pattern launched PYRIT_B200_HOT_PATTERN times gets its
    specialised kernel compiled in the background (the runtime kernel serves until then); a
    pattern used fewer times never compiles."""
    import subprocess
    import sys
    import textwrap
    script = textwrap.dedent("""
        import numpy as np, torch
        import paper_1709_00178_b200 as P
        from paper_1709_00178_b200 import _lib as L
        code = P.CodeSpec(10, 4, P.FieldSpec.gf256_r17())
        d = torch.from_numpy(np.random.default_rng(5).integers(0, 256, (14, 8 * 16 * 512), dtype=np.uint8)).cuda()
        d[10:] = P.encode(d[:10], code)
        ref = d.clone()
        kernels = []
        for er in [(2, 3, 4, 5)] * 3 + [(0, 2, 7, 11)] * 4:
            d[list(er)] = 0
            P.decode(d, er, code)
            torch.cuda.synchronize()
            assert torch.equal(d, ref)
            kernels.append(P.Plan.last_launch()["kernel"])
        cold = L.load().pyrit_jit_compiles()
        L.check(L.load().pyrit_jit_wait())
        d[[0, 2, 7, 11]] = 0
        P.decode(d, (0, 2, 7, 11), code)
        torch.cuda.synchronize()
        assert torch.equal(d, ref)
        kernels.append(P.Plan.last_launch()["kernel"])
        print(cold, L.load().pyrit_jit_compiles(), " ".join(kernels))
    """)
    env = dict(os.environ, PYRIT_B200_TIERED="1", PYRIT_B200_JIT_CACHE=str(tmp_path), PYRIT_B200_HOT_PATTERN="4")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, cwd=root,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.split()
    kernels = out[2:]
    assert all(k.startswith("pyrit_ring_rt_") for k in kernels[:7]), kernels
    assert kernels[-1].startswith("pyrit_ring_k10_e4_w8_n17"), kernels  # the hot pattern, specialised
    assert int(out[1]) == 1  # one compile: the pattern used 4 times, not the one used 3 times


@pytest.mark.parametrize("f", [G256, G4096], ids=lambda f: f"w{f.w}n{f.n}")
def test_apply_ringmat_on_device(cuda, f):
    """pyrit_cu_apply_ringmat (SURVEY 8(b)'s operator with the ring matrix as operand): raw
    masks, non-canonical ones included, on the runtime kernel with no compile; on a strip
    the runtime kernel cannot take (8-byte aligned) the compiled program of the field matrix
    gives the same symbols."""
    import torch
    rng = np.random.default_rng(17)
    e, k = 4, 12
    m = rng.integers(0, 1 << f.w, (e, k), dtype=np.uint16)
    reps = np.array([[P.sparse_transform(int(x), f) ^ (f.modulus if (i + j) % 3 == 0 else 0)
                      for j, x in enumerate(row)] for i, row in enumerate(m)], dtype=np.uint32)
    lib = L.load()
    for strip in (4096 + 64, 4096 + 8):
        data = rand_symbols(k, f.w * strip, strip)
        d = torch.from_numpy(data).to(cuda)
        out = torch.zeros((e, f.w * strip), dtype=torch.uint8, device=cuda)
        jit0 = lib.pyrit_jit_compiles()
        P.apply_ringmat(f, reps, [d[j].data_ptr() for j in range(k)], [out[i].data_ptr() for i in range(e)], strip)
        torch.cuda.synchronize()
        if strip % 16 == 0:
            rt_launched()
            assert lib.pyrit_jit_compiles() == jit0
        np.testing.assert_array_equal(out.cpu().numpy(), oracle_ring(f, m, data))


def test_warmup_loads_every_geometry(cuda):
    """pyrit_warmup loads the runtime-matrix modules of all five ring geometries; decoding after
    it still repairs (and compiles nothing)."""
    import torch
    lib = L.load()
    L.check(lib.pyrit_warmup(cuda.index or 0))
    wl = WORKLOADS[2]
    ss = wl.fld.w * 16 * 64
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    full = torch.from_numpy(np.concatenate([data, oracle_ring(wl.fld, P.cauchy_parity_matrix(wl.code), data)])).to(cuda)
    ref = full.clone()
    jit0 = lib.pyrit_jit_compiles()
    full[[2, 11]] = 0
    P.decode(full, (2, 11), wl.code)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)
    assert lib.pyrit_jit_compiles() == jit0


@pytest.mark.parametrize("f", [G256, G4096], ids=lambda f: f"w{f.w}n{f.n}")
def test_planned_launches_rebind_to_new_buffers(cuda, f):
    """The planner's result (op lists, parts, pair cases) is kept per program and thread;
    the same program on other buffers, another window or after another program only gets
    new tensor maps and output bases (runtime.cpp bind_ring_rt).  Alternate two programs
    over two buffer sets and two windows; every result against the oracle."""
    rng = np.random.default_rng(100 + f.w)
    k, e = 7, 4
    strip = 16 * 520
    ss = f.w * strip
    mats = [rng.integers(1, 1 << f.w, (e, k), dtype=np.uint16) for _ in range(2)]
    plans = [P.Plan.create(f, m) for m in mats]
    datas = [rand_symbols(k, ss, 40 + i) for i in range(2)]
    wants = [[oracle_ring(f, m, d) for d in datas] for m in mats]
    with mode(4):
        for step, (pi, di, win) in enumerate([(0, 0, None), (1, 0, None), (0, 1, None), (1, 1, (16 * 9, 16 * 200)),
                                              (0, 0, (0, 16 * 131)), (0, 1, None), (1, 0, None)]):
            off, length = win if win else (0, strip)
            init = rand_symbols(e, ss, 60 + step)
            got = run_plan(cuda, plans[pi], datas[di], e, strip, off, length, init=init)
            rt_launched()
            exp = init.copy()
            for i in range(e):
                for s in range(f.w):
                    a = s * strip + off
                    exp[i, a:a + length] = wants[pi][di][i, a:a + length]
            np.testing.assert_array_equal(got, exp, err_msg=f"step {step}")


def test_launch_shapes(cuda):
    """The shapes the planner picks (runtime.cpp build_ring_rt): one output -> one 256-thread
    part; two -> two 128-thread parts; three or more -> four parts plus the 128-thread
    producer warp group that issues the TMA copies (640 threads, setmaxnreg in ring_rt.cuh)."""
    f = G256
    rng = np.random.default_rng(5)
    k, strip = 6, 16 * 256
    data = rand_symbols(k, f.w * strip, 77)
    with mode(4):
        for e, threads in [(1, 256), (2, 256), (3, 640), (4, 640)]:
            m = rng.integers(1, 1 << f.w, (e, k), dtype=np.uint16)
            got = run_plan(cuda, P.Plan.create(f, m), data, e, strip)
            rt_launched()
            assert P.Plan.last_launch()["threads"] == threads, (e, P.Plan.last_launch())
            np.testing.assert_array_equal(got, oracle_ring(f, m, data))

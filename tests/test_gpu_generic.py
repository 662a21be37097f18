"""The generic bit-matrix kernel and tiered compilation (GPU).

The generic kernel (kernels.cu) evaluates any compiled program's GF(2) bitmatrix with no per-code
compilation. It serves the first launches of a code whose specialised kernel is still being
compiled in the background (tiered compilation), and every launch in kernel mode 3. Kernel mode 3
makes it cheap to run the reference's acceptance criterion 5 here (acceptance.cpp:142-194):
- every erasure pattern of weight <= r for (4,2) and (6,3) over GF(2^4) and (6,3) over GF(2^6),
  both transforms;
- random patterns for the production-size codes.
Each distinct pattern would otherwise be its own generated kernel.
"""
from __future__ import annotations

import itertools
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from paper_1709_00178_b200 import _lib as L
from tests.helpers import G16, G64, ofield

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture
def generic(cuda):
    lib = L.load()
    L.check(lib.pyrit_set_kernel_mode(3))
    yield
    L.check(lib.pyrit_set_kernel_mode(0))


def _roundtrip(cuda, code, data, erased):
    import torch
    d = torch.from_numpy(data).to(cuda)
    parity = P.encode(d, code)
    full = torch.cat([d, parity])
    ref = full.clone()
    full[list(erased)] = 0
    P.decode(full, list(erased), code)
    torch.cuda.synchronize()
    return parity, bool(torch.equal(full, ref))


def test_generic_encode_matches_oracle_all_small_codes(cuda, generic):
    """acceptance.cpp:197-222 (criterion 6) on the generic kernel: every (k, r) <= 5 over GF(2^4) and
    GF(2^6), both transforms, against the field oracle."""
    rng = np.random.default_rng(600)
    for f in (G16, G64):
        for k in range(1, 6):
            for r in range(1, 6):
                for kind in (0, 1):
                    code = P.CodeSpec(k, r, f, P.TransformKind(kind))
                    strip = 32
                    data = rng.integers(0, 256, (k, f.w * strip), dtype=np.uint8)
                    want = np.stack(O.apply_columns(ofield(f), P.cauchy_parity_matrix(code), list(data), strip,
                                                    kind=kind))
                    parity, ok = _roundtrip(cuda, code, data, range(min(r, k)))
                    assert np.array_equal(parity.cpu().numpy(), want), (f.w, k, r, kind)
                    assert ok
                    assert P.Plan.last_launch()["kernel"] == "pyrit_generic_bitmatrix"


def test_acceptance_criterion5_every_small_pattern(cuda, generic):
    """acceptance.cpp:150-170: every erasure pattern of weight <= r, (4,2)/(6,3) GF(2^4), (6,3) GF(2^6),
    both transforms."""
    rng = np.random.default_rng(500)
    patterns = 0
    for k, r, f in ((4, 2, G16), (6, 3, G16), (6, 3, G64)):
        for kind in (0, 1):
            code = P.CodeSpec(k, r, f, P.TransformKind(kind))
            data = rng.integers(0, 256, (k, f.w * 64), dtype=np.uint8)
            for weight in range(1, r + 1):
                for erased in itertools.combinations(range(k + r), weight):
                    _, ok = _roundtrip(cuda, code, data, erased)
                    assert ok, (k, r, f.w, kind, erased)
                    patterns += 1
    assert patterns == 2 * (21 + 129 + 129)  # 558, as acceptance.cpp counts them


def test_acceptance_criterion5_production_codes(cuda, generic):
    """acceptance.cpp:172-193: random patterns of weight 1..r for (8,4) GF(2^4) embedding, (40,20)
    GF(2^6) embedding, (20,40) GF(2^6) parity (the paper's codes), 1000 each: with the 558 above, the
    reference's 3558 patterns."""
    rng = np.random.default_rng(501)
    for k, r, f, kind, rounds in ((8, 4, G16, 0, 1000), (40, 20, G64, 0, 1000), (20, 40, G64, 1, 1000)):
        code = P.CodeSpec(k, r, f, P.TransformKind(kind))
        data = rng.integers(0, 256, (k, f.w * 64), dtype=np.uint8)
        for _ in range(rounds):
            weight = 1 + int(rng.integers(0, r))
            erased = sorted(rng.permutation(k + r)[:weight].tolist())
            _, ok = _roundtrip(cuda, code, data, erased)
            assert ok, (k, r, kind, erased)


def test_generic_baseline_shapes_and_batches(cuda, generic):
    """The BASELINE codes (reduced strips), stripe batches and column windows on the generic kernel."""
    import torch
    from paper_1709_00178_b200.workloads import WORKLOADS
    for cfg in (1, 2, 3, 5):
        wl = WORKLOADS[cfg]
        f = wl.fld
        strip = 16 * 257
        nb = 3
        rng = np.random.default_rng(cfg)
        data = rng.integers(0, 256, (nb, wl.k, f.w * strip), dtype=np.uint8)
        m = P.cauchy_parity_matrix(wl.code)
        plan = P.Plan.encode(wl.code)
        d = torch.from_numpy(data).to(cuda)
        out = torch.full((nb, wl.m, f.w * strip), 0x55, dtype=torch.uint8, device=cuda)
        sym = f.w * strip
        off, length = 16, strip - 48
        plan.apply_batch([d[0, j].data_ptr() for j in range(wl.k)], [out[0, i].data_ptr() for i in range(wl.m)],
                         strip, nb, wl.k * sym, wl.m * sym, off, length,
                         stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert P.Plan.last_launch()["kernel"] == "pyrit_generic_bitmatrix"
        got = out.cpu().numpy()
        for b in range(nb):
            want = O.ring_replay(ofield(f), m, [data[b, j].copy() for j in range(wl.k)], strip, off=off,
                                 length=length, outs=[np.full(sym, 0x55, dtype=np.uint8) for _ in range(wl.m)])
            for i in range(wl.m):
                assert np.array_equal(got[b, i], want[i]), (cfg, b, i)


@pytest.mark.parametrize("rt", ["1", "0"])
def test_tiered_compilation(cuda, tmp_path, rt):
    """A code with no prebuilt or cached kernel: the first launch runs the runtime-matrix ring kernel
    (PYRIT_B200_RT=0: the generic bit-matrix kernel) while the specialised one compiles in the
    background; after pyrit_jit_wait() the next launch runs the specialised kernel. Both give the
    oracle's bytes."""
    script = textwrap.dedent("""
        import time, numpy as np, torch
        import oracle as O
        import paper_1709_00178_b200 as P
        from paper_1709_00178_b200 import _lib as L
        f = P.FieldSpec.aop(10)
        code = P.CodeSpec(7, 3, f)
        strip = 4096
        data = np.random.default_rng(9).integers(0, 256, (7, 10 * strip), dtype=np.uint8)
        want = np.stack(O.ring_replay(O.Field(10, 11, 0, 1, 10, 0x7FF), P.cauchy_parity_matrix(code), list(data), strip))
        d = torch.from_numpy(data).cuda()
        kernels, ok = [], []
        p = P.encode(d, code)
        torch.cuda.synchronize()
        kernels.append(P.Plan.last_launch()["kernel"])
        ok.append(bool(np.array_equal(p.cpu().numpy(), want)))
        L.check(L.load().pyrit_jit_wait())  # the background compile is done: the next launch is specialised
        for attempt in range(60):
            p = P.encode(d, code)
            torch.cuda.synchronize()
            kernels.append(P.Plan.last_launch()["kernel"])
            ok.append(bool(np.array_equal(p.cpu().numpy(), want)))
            if kernels[-1] != "pyrit_generic_bitmatrix" and not kernels[-1].startswith("pyrit_ring_rt_"):
                break
            time.sleep(0.5)
        print(kernels[0], kernels[1], all(ok), L.load().pyrit_jit_compiles())
    """)
    env = dict(os.environ, PYRIT_B200_TIERED="1", PYRIT_B200_JIT_CACHE=str(tmp_path), PYRIT_B200_RT=rt)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    first, second, ok, jit = r.stdout.split()[-4:]
    # the launch right after pyrit_jit_wait() already runs the specialised kernel
    stand_in = "pyrit_ring_rt_w10_n11" if rt == "1" else "pyrit_generic_bitmatrix"
    assert first == stand_in and second.startswith("pyrit_ring_k"), r.stdout
    assert ok == "True" and int(jit) == 1


def test_exit_while_compiling(cuda, tmp_path):
    """A process may exit while a background compile is still running: it must exit cleanly (the
    compile state is never destroyed under the running thread) and promptly."""
    script = textwrap.dedent("""
        import numpy as np, torch
        import paper_1709_00178_b200 as P
        code = P.CodeSpec(11, 5, P.FieldSpec.aop(12))
        d = torch.from_numpy(np.random.default_rng(3).integers(0, 256, (11, 12 * 4096), dtype=np.uint8)).cuda()
        p = P.encode(d, code)
        torch.cuda.synchronize()
        print(P.Plan.last_launch()["kernel"])
    """)
    env = dict(os.environ, PYRIT_B200_TIERED="1", PYRIT_B200_JIT_CACHE=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, cwd=ROOT,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split()[-1] == "pyrit_ring_rt_w12_n13"

"""Large codes and the on-disk JIT cache (GPU).

Programs with no prebuilt cubin are generated and compiled with NVRTC on first use. Each
compiled cubin is kept under PYRIT_B200_JIT_CACHE, so a second process loads it without
compiling. This file also runs a code far beyond the BASELINE shapes: (64, 32) over GF(2^12),
116k XORs per column word, split into output parts.
"""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import oracle as O
import paper_1709_00178_b200 as P
from tests.helpers import ofield

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_jit_cache_persists_across_processes(cuda, tmp_path):
    script = textwrap.dedent("""
        import numpy as np, torch
        import paper_1709_00178_b200 as P
        from paper_1709_00178_b200 import _lib as L
        code = P.CodeSpec(9, 3, P.FieldSpec.aop(10))   # no prebuilt cubin for this program
        d = torch.from_numpy(np.random.default_rng(1).integers(0, 256, (9, 10 * 4096), dtype=np.uint8)).cuda()
        p = P.encode(d, code)
        torch.cuda.synchronize()
        print(L.load().pyrit_jit_compiles(), int(P.digest(p).item()))
    """)
    env = dict(os.environ, PYRIT_B200_JIT_CACHE=str(tmp_path))
    runs = [subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, cwd=ROOT,
                           timeout=600) for _ in range(2)]
    for r in runs:
        assert r.returncode == 0, r.stderr[-2000:]
    (n1, d1), (n2, d2) = (r.stdout.split()[-2:] for r in runs)
    assert int(n1) >= 1 and int(n2) == 0 and d1 == d2
    assert list(tmp_path.glob("pyrit_ring_*.cubin"))


@pytest.mark.gpu
def test_large_code_encode_and_repair(cuda):
    import torch
    f = P.FieldSpec.aop(12)
    k, r = 64, 32
    code = P.CodeSpec(k, r, f)
    strip = 16 * 1024
    ss = f.w * strip
    data = np.random.default_rng(64).integers(0, 256, (k, ss), dtype=np.uint8)
    m = P.cauchy_parity_matrix(code)
    want = np.stack(O.ring_replay(ofield(f), m, list(data), strip))
    d = torch.from_numpy(data).to(cuda)
    parity = P.encode(d, code)
    torch.cuda.synchronize()
    assert np.array_equal(parity.cpu().numpy(), want)
    full = torch.cat([d, parity])
    ref = full.clone()
    erased = [3, 40, 63, 70]
    full[erased] = 0
    P.decode(full, erased, code)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("f,k,r,kind", [
    (P.FieldSpec.gf16_aop(), 12, 4, 0), (P.FieldSpec.gf16_aop(), 8, 8, 0), (P.FieldSpec.gf16_aop(), 4, 12, 1),
    (P.FieldSpec.gf64_esp(), 48, 16, 0), (P.FieldSpec.gf64_esp(), 16, 48, 1)])
def test_maximum_length_codes(cuda, f, k, r, kind):
    """k + r = 2^w, the largest code each field admits (matrix.hpp:27-30): encode, and decode of r
    erasures spread over data and parity."""
    import torch
    code = P.CodeSpec(k, r, f, P.TransformKind(kind))
    strip = 16 * 300
    data = np.random.default_rng(k * 100 + r).integers(0, 256, (k, f.w * strip), dtype=np.uint8)
    m = P.cauchy_parity_matrix(code)
    want = np.stack(O.ring_replay(ofield(f), m, list(data), strip, kind=kind))
    d = torch.from_numpy(data).to(cuda)
    parity = P.encode(d, code)
    torch.cuda.synchronize()
    assert np.array_equal(parity.cpu().numpy(), want)
    full = torch.cat([d, parity])
    ref = full.clone()
    erased = sorted(np.random.default_rng(r).choice(k + r, size=r, replace=False).tolist())
    full[erased] = 0
    P.decode(full, erased, code)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)

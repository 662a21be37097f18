"""Negative control: the parity checks can fail.  The reference ships one (`pyrit verify
--inject-theta-fault`, tools/pyrit.cpp:281-282, selfcheck.hpp:28-34: one bit of the embedding
idempotent flipped); here pyrit_plan_inject_fault flips one bit of one ring representative of a
compiled plan, and the same comparison against the oracle that every parity test makes must then
report a mismatch -- on the CPU interpreter and on the GPU (runtime-matrix and generated kernels)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1709_00178_b200 as P
from paper_1709_00178_b200 import _lib as L
from paper_1709_00178_b200.workloads import WORKLOADS
from tests.helpers import oracle_ring, seeded_symbols


def _case(cfg):
    wl = WORKLOADS[cfg]
    ss = wl.fld.w * 16 * 200
    data = seeded_symbols(wl.k, ss, wl.fld.w, wl.seed)
    C = P.cauchy_parity_matrix(wl.code)
    return wl, ss, data, C, oracle_ring(wl.fld, C, data)


@pytest.mark.parametrize("cfg", [2, 5])
def test_fault_detected_by_interpreter(cfg):
    wl, ss, data, C, want = _case(cfg)
    plan = P.Plan.create(wl.fld, C)
    clean = np.stack(plan.interpret(list(data), ss // wl.fld.w))
    np.testing.assert_array_equal(clean, want)  # the control: clean plan agrees
    plan.inject_fault(5, 1)
    bad = np.stack(plan.interpret(list(data), ss // wl.fld.w))
    assert not np.array_equal(bad, want), "an injected fault went undetected"
    # the fault lands in output row 5 // k only
    row = 5 // wl.k
    assert not np.array_equal(bad[row], want[row])
    for i in range(wl.m):
        if i != row:
            np.testing.assert_array_equal(bad[i], want[i])


def test_fault_rejects_bad_arguments():
    wl = WORKLOADS[2]
    plan = P.Plan.create(wl.fld, P.cauchy_parity_matrix(wl.code))
    with pytest.raises(P.PyritError):
        plan.inject_fault(10_000, 0)
    with pytest.raises(P.PyritError):
        plan.inject_fault(0, wl.fld.n)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [4, 0])
@pytest.mark.parametrize("cfg", [2, 5])
def test_fault_detected_on_gpu(cuda, cfg, mode):
    """mode 4: the runtime-matrix kernel reads the faulty representative at launch; mode 0: the
    faulty program compiles to its own specialised kernel (NVRTC).  Either way the GPU output
    must stop matching the oracle."""
    import torch
    wl, ss, data, C, want = _case(cfg)
    lib = L.load()
    d = torch.from_numpy(data).to(cuda)
    out = torch.zeros((wl.m, ss), dtype=torch.uint8, device=cuda)

    def run(plan):
        out.zero_()
        plan.apply([d[j].data_ptr() for j in range(wl.k)], [out[i].data_ptr() for i in range(wl.m)], ss // wl.fld.w)
        torch.cuda.synchronize()
        return out.cpu().numpy(), P.Plan.last_launch()["kernel"]

    L.check(lib.pyrit_set_kernel_mode(mode))
    try:
        plan = P.Plan.create(wl.fld, C)
        got, k_clean = run(plan)
        np.testing.assert_array_equal(got, want)
        plan.inject_fault(5, 1)
        bad, k_bad = run(plan)
    finally:
        L.check(lib.pyrit_set_kernel_mode(0))
    assert not np.array_equal(bad, want), "GPU parity check missed an injected fault"
    if mode == 4:
        assert k_bad.startswith("pyrit_ring_rt_")
    else:
        assert k_bad != k_clean  # a different program, a different kernel

"""Generate tests/golden/ fixtures by running the REFERENCE itself.

    python tests/golden/make_golden.py      (needs /root/reference, build container only)

Everything here comes out of oracle/_ref/libpyrit_ref.so -- the unmodified
reference headers compiled in place (oracle/Makefile) -- so the fixtures pin
both the C oracle and the GPU path to the reference's own outputs:

  * Cauchy parity matrices, ring representatives and schedule statistics for
    every BASELINE field (the reference cannot build GF(2^8)/R_{2,17} ring
    schedules correctly, so for that field only the field-level outputs are
    recorded, plus its CRS/oracle_apply parity);
  * parity bytes for each BASELINE configuration at a reduced fragment size,
    from the reference's encode() (ring) or, for R_{2,17}, encode_crs() and
    oracle_apply(); the data bytes are regenerated from the seed by
    oracle.fill_np (counter-based, see pyrit_oracle.c or_fill);
  * decode results (the reference's decode() for AOP/ESP fields; decode_matrix
    for R_{2,17});
  * small GF16/GF64 codes for both transforms (test_codec.cpp:53-80 grid).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

CONFIGS = {
    1: (O.GF16, 4, 2, 0),
    2: (O.GF256_R17, 10, 4, 1),
    3: (O.GF1024, 12, 4, 2),
    4: (O.GF256_R17, 10, 4, 3),
    5: (O.GF4096, 16, 4, 4),
}
STRIP = 96  # bytes per strip in the fixtures (a multiple of 16 and of 8)


def data_for(f, k, seed, strip=STRIP):
    ss = f.w * strip
    return np.stack([O.fill_np(seed, j, ss) for j in range(k)])


def main():
    assert os.path.isdir("/root/reference/proj/include/pyrit"), "needs the reference tree"
    O.build()
    meta = {"generator": "tests/golden/make_golden.py", "strip_bytes": STRIP, "configs": {}}
    arrays = {}
    for cfg, (f, k, r, seed) in CONFIGS.items():
        c = O.ref_cauchy(k, r, f)
        entry = {"k": k, "r": r, "w": f.w, "n": f.n, "modulus": f.modulus, "seed": seed,
                 "cauchy": c.tolist()}
        ring_ok = f.n <= 16  # RingElem is uint16 (field.hpp:12)
        if ring_ok:
            entry["reps"] = [[O.ref_sparse_transform(int(u), f) for u in row] for row in c]
            entry["schedule_stats"] = O.ref_schedule_stats(f, c)
            entry["schedule_stats_dense"] = O.ref_schedule_stats(f, c, rep=1)
        entry["crs_stats"] = O.ref_schedule_stats(f, c, crs=1)
        data = data_for(f, k, seed)
        ss = data.shape[1]
        flat = np.ascontiguousarray(data.reshape(-1))
        if ring_ok:
            parity = O.ref_encode(f, k, r, flat, ss).reshape(r, ss)
        else:
            parity = O.ref_encode(f, k, r, flat, ss, crs=1).reshape(r, ss)
        plain = O.ref_oracle_apply(f, c, flat, ss).reshape(r, ss)
        assert np.array_equal(parity, plain), cfg
        arrays[f"cfg{cfg}_parity"] = parity
        if cfg == 4:
            erased = [1, 6, 9, 10]
            surv = [i for i in range(k + r) if i not in erased][:k]
            from ctypes import byref, c_uint, c_uint16, c_uint32
            out = (c_uint16 * (k * k))()
            rows = c_uint()
            sv = (c_uint32 * k)(*surv)
            rc = O.ref().ref_decode_matrix(k, r, f.w, f.n, f.modulus, sv, out, byref(rows))
            assert rc == 0
            entry["decode_erased"] = erased
            entry["decode_survivors"] = surv
            entry["decode_matrix"] = np.frombuffer(bytes(out), dtype=np.uint16)[: rows.value * k].reshape(
                rows.value, k).tolist()
        if ring_ok:
            full = np.concatenate([data, parity])
            work = np.ascontiguousarray(full.copy())
            erased = list(range(min(k, r)))
            work[erased] = 0xAA
            O.ref_decode(f, k, r, work.reshape(-1), ss, erased)
            assert np.array_equal(work, full)
            entry["decode_roundtrip_erased"] = erased
        meta["configs"][str(cfg)] = entry

    # small codes, both transforms (test_codec.cpp:53-80)
    small = []
    rng = np.random.default_rng(101)
    for f in (O.GF16, O.GF64):
        for k in range(1, 6):
            for r in range(1, 6):
                for transform in (0, 1):
                    ss = int(np.lcm(f.w, 8)) * 2
                    data = rng.integers(0, 256, (k, ss), dtype=np.uint8)
                    p = O.ref_encode(f, k, r, np.ascontiguousarray(data.reshape(-1)), ss, transform=transform)
                    key = f"small_w{f.w}_k{k}_r{r}_t{transform}"
                    arrays[key + "_data"] = data
                    arrays[key + "_parity"] = p.reshape(r, ss)
                    small.append(key)
    meta["small"] = small
    # field KATs straight from the reference: all sparse reps of GF16/GF64/GF1024/GF4096
    meta["sparse_reps"] = {str(f.w): [O.ref_sparse_transform(u, f) for u in range(1 << f.w)]
                           for f in (O.GF16, O.GF64, O.GF1024, O.GF4096)}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=None, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"), os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()

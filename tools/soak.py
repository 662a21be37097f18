#!/usr/bin/env python
"""Randomised soak of the generated kernels (validation aid, not a unit test).

    python tools/soak.py [--cases 300] [--seed 1]

Each case draws a field, code shape, transform, strip length / alignment, stripe
batch, kernel mode and staged producer (cp.async, TMA tensor, TMA + producer
warp), launches one stripe batch through the C ABI and compares every output
byte with the C oracle's ring replay.  Prints one JSON summary line.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time
os.environ.setdefault("PYRIT_B200_TIERED", "0")  # measure/validate the specialised kernels, never the generic stand-in

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--knobs", action="store_true",
                    help="also random matrices, more (w, n, p) fields and random compile knobs (parts, fragment "
                         "groups, pair sharing windows, CTA size)")
    ap.add_argument("--rt", action="store_true",
                    help="runtime-matrix ring kernel only (kernel mode 4): random matrices over the AOT ring "
                         "geometries, 16-byte aligned strips, e up to 24 outputs, k up to 64")
    a = ap.parse_args()

    import numpy as np
    import torch

    import oracle as O
    import paper_1709_00178_b200 as P
    from paper_1709_00178_b200 import _lib as L

    dev = torch.device("cuda", 0)
    lib = L.load()
    rng = random.Random(a.seed)
    fields = [P.FieldSpec.gf16_aop(), P.FieldSpec.gf64_esp(), P.FieldSpec.gf256_r17(), P.FieldSpec.aop(10),
              P.FieldSpec.aop(12)]
    exotic = [P.FieldSpec(2, 3, 0, 1, 2, 0b111), P.FieldSpec(3, 7, 0, 1, 3, 0b1011),
              P.FieldSpec(4, 15, 0, 1, 4, 0b10011)]
    knob_names = ("PARTS", "PART_GROUP", "PART_CSE", "CSE_WINDOW", "THREADS")
    fails, t0, kernels, rt_cases = [], time.time(), set(), 0
    for case in range(a.cases):
        f = rng.choice(fields + (exotic if a.knobs else []))
        k = rng.randint(1, min(64 if a.rt else 32, f.field_size() - 1))
        r = rng.randint(1, min(24 if a.rt else 16, f.field_size() - k))
        kind = rng.choice([0, 0, 0, 1]) if f not in exotic else 0
        strip = 16 * rng.randint(1, 2048) + (0 if a.rt else rng.choice([0, 0, 0, 4, 8]))
        nb = rng.choice([1, 1, 2, 5])
        mode = 4 if a.rt else rng.choice([0, 2, 2])
        prod = rng.choice(["1", "2", "2", "3"])
        os.environ["PYRIT_B200_COPY"] = "1" if prod == "1" else "2"
        os.environ["PYRIT_B200_WS"] = "1" if prod == "3" else "0"
        L.check(lib.pyrit_set_kernel_mode(mode))
        code = P.CodeSpec(k, r, f, P.TransformKind(kind))
        knobs = {}
        if a.knobs:
            knobs = {"PARTS": rng.choice([1, 2, 4]), "PART_GROUP": rng.randint(1, 4), "PART_CSE": rng.randint(0, 1),
                     "CSE_WINDOW": rng.choice([0, 1, 3, 9]), "THREADS": rng.choice([256, 512])}
        for n in knob_names:
            os.environ.pop("PYRIT_B200_" + n, None)
        for n, v in knobs.items():
            os.environ["PYRIT_B200_" + n] = str(v)
        if (a.knobs or a.rt) and rng.random() < 0.5:
            m = np.array([[rng.randrange(f.field_size()) for _ in range(k)] for _ in range(r)], dtype=np.uint16)
        else:
            m = P.cauchy_parity_matrix(code)
        plan = P.Plan.create(f, m, P.TransformKind(kind))
        sym = f.w * strip
        data = np.random.default_rng(case).integers(0, 256, (nb, k, sym), dtype=np.uint8)
        d = torch.from_numpy(data).to(dev)
        out = torch.full((nb, r, sym), 0x33, dtype=torch.uint8, device=dev)
        try:
            plan.apply_batch([d[0, j].data_ptr() for j in range(k)], [out[0, i].data_ptr() for i in range(r)], strip,
                             nb, k * sym, r * sym, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            kernels.add(P.Plan.last_launch()["kernel"])
            rt_cases += P.Plan.last_launch()["kernel"].startswith("pyrit_ring_rt_")
            got = out.cpu().numpy()
            of = O.Field(f.w, f.n, f.kind, f.s, f.r_esp, f.modulus)
            for b in sorted({0, nb - 1}):
                want = O.ring_replay(of, m, [data[b, j].copy() for j in range(k)], strip, kind=kind)
                if not all(np.array_equal(got[b, i], want[i]) for i in range(r)):
                    fails.append({"case": case, "field": [f.w, f.n], "k": k, "r": r, "kind": kind, "strip": strip,
                                  "nb": nb, "mode": mode, "producer": prod, "stripe": b, "knobs": knobs,
                                  "kernel": P.Plan.last_launch()["kernel"]})
                    break
        except Exception as e:  # report, keep soaking
            fails.append({"case": case, "error": str(e)[:200], "k": k, "r": r, "strip": strip, "producer": prod})
        plan.close()
    L.check(lib.pyrit_set_kernel_mode(0))
    for n in knob_names:
        os.environ.pop("PYRIT_B200_" + n, None)
    print(json.dumps({"cases": a.cases, "knobs": a.knobs, "rt": a.rt, "failures": len(fails), "distinct_kernels": len(kernels), "runtime_matrix_cases": rt_cases,
                      "seconds": round(time.time() - t0, 1), "first_failures": fails[:5]}))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())

"""Generate the dispatch blocks of the runtime-matrix ring kernel (csrc/ring_rt.cu).

    python -m paper_1709_00178_b200.gen_ring_rt <out.inc> [pair distance]

For every kernel instance (w, n, E outputs, V words per thread, transform) this
emits RtOps<...>::run(q, d, acc, x): one inline-PTX block whose `brx.idx` jumps
through a table of E*(D+1)*n targets; target c = (i*(D+1) + ds)*n + sh XORs the
input strips, rotated by sh ring positions (ds = 0) or by sh and sh+ds (a
paired-shift case, rows reached by both with one 3-input LOP3), into the
accumulators of output i (schedule.hpp:132-161: ring row t of output i
accumulates input strip (t - sh) mod n).  Every register index inside a case is
fixed, so the runtime matrix never indexes registers dynamically, and the jump
is warp-uniform.  D = pair_d(w, n, v, PYRIT_RT_PAIR_D) (csrc/kernels.hpp rt_pair_d).
The instance list (FIELDS) must match PYRIT_RT_FIELDS in csrc/ring_rt.cu.
"""
from __future__ import annotations

import sys

# (w, n) of the ahead-of-time instances; ring_rt.cu lists the moduli
FIELDS = [(4, 5), (6, 9), (8, 17), (10, 11), (12, 13)]


def part_outputs(n: int, w: int, v: int) -> int:  # kernels.hpp rt_part_outputs
    return max(1, min(8, (104 - 4 * w) // (4 * n) if v == 4 else 36 // n))


def instances():
    for w, n in FIELDS:
        for v in (2, 4):
            for e in range(1, part_outputs(n, w, v) + 1):
                for par in (False, True):
                    yield w, n, e, v, par


def pair_d(w: int, n: int, v: int, d: int, aop_all: bool = True) -> int:  # kernels.hpp rt_pair_d
    """Paired-shift cases exist for the V = 4 instances only (the single-output
    V = 2 shape is HBM-bound without them): distances up to d, or every distance
    in the all-one-polynomial fields (w = n-1), where any pair overlaps in w-1 rows."""
    if v != 4 or d == 0:
        return 0
    return (n - 1) // 2 if (aop_all and w + 1 == n) else min(d, (n - 1) // 2)


def emit(w: int, n: int, e: int, v: int, par: bool, dmax: int = 0, aop_all: bool = True) -> str:
    """RtOps<...>::run(q, d, acc, x): threaded dispatch of one op list (bytes
    c = (i*(D+1) + ds)*n + sh, terminated by e*(D+1)*n) read from shared memory at
    q, with d the op already loaded.  ds = 0 is the single shift sh; ds = 1..D is
    the pair of shifts (sh, sh+ds) of one representative as ONE case: a ring row
    both shifts reach takes one 3-input `lop3 0x96` instead of two XORs.  Every case
    ends with the jump to the next op: the op after it is loaded one case ahead, so a case costs its XORs plus a move, a byte load, an
    add and the indexed jump.  The lists of one part lie back to back, so on
    return (at the sentinel) d already holds the first op of the next input's list
    and the next call jumps without waiting on shared memory."""
    ar = w if par else n  # accumulator rows
    xr = n if par else w  # input rows in registers
    nacc = e * ar * v

    def acc(i, r, l):
        return (i * ar + r) * v + l

    def xop(t, l):
        return nacc + 2 + t * v + l

    qop = nacc  # "+r"(q), "+r"(d) follow the accumulators
    dop = nacc + 1
    xbase = nacc + 2
    lines = []
    targets = []
    dd = pair_d(w, n, v, dmax, aop_all)
    for c in range(e * (dd + 1) * n):
        ids, sh = divmod(c, n)
        i, ds = divmod(ids, dd + 1)
        body = [f"mov.b32 c, %{dop}; ld.shared.u8 %{dop}, [%{qop}]; add.u32 %{qop}, %{qop}, 1;"]
        for r in range(ar):
            # input strips that land on accumulator row r: (r - sh) and, for a pair, (r - sh - ds) mod n
            ts = [t for t in {(r - sh) % n, (r - sh - ds) % n} if t < xr] if ds else [t for t in [(r - sh) % n] if t < xr]
            ts.sort()
            for l in range(v):
                a = acc(i, r, l)
                if len(ts) == 1:
                    body.append(f"xor.b32 %{a}, %{a}, %{xop(ts[0], l)};")
                elif len(ts) == 2:
                    body.append(f"lop3.b32 %{a}, %{a}, %{xop(ts[0], l)}, %{xop(ts[1], l)}, 0x96;")
        body.append("brx.idx.uni c, T;")
        lab = f"L{c}"
        targets.append(lab)
        lines.append(f'"{lab}: ' + " ".join(body) + '\\n"')
    targets.append("LX")
    outs = ", ".join(f'"+r"(acc[{i}][{r}][{l}])' for i in range(e) for r in range(ar) for l in range(v))
    ins = ", ".join(f'"r"(x[{t}][{l}])' for t in range(xr) for l in range(v))
    tpl = f"{w}, {n}, {e}, {v}, {'true' if par else 'false'}"
    s = [f"static_assert(rt_pair_d({w}, {n}, {v}) == {dd}, \"gen_ring_rt.py pair_d and kernels.hpp rt_pair_d disagree\");",
         f"template <> struct RtOps<{tpl}> {{"]
    s.append(f"  static __device__ __forceinline__ void run(u32& q, u32& d, u32 (&acc)[{e}][{ar}][{v}], "
             f"const u32 (&x)[{xr}][{v}]) {{")
    s.append('    asm volatile("{\\n .reg .b32 c;\\n"')
    s.append(f'      "mov.b32 c, %{dop}; ld.shared.u8 %{dop}, [%{qop}]; add.u32 %{qop}, %{qop}, 1;\\n"')
    s.append(f'      "T: .branchtargets {", ".join(targets)};\\n"')
    s.append('      "brx.idx.uni c, T;\\n"')
    for ln in lines:
        s.append("      " + ln)
    s.append('      "LX:\\n}\\n"')
    s.append(f'      : {outs}, "+r"(q), "+r"(d)')
    s.append(f'      : {ins}')
    s.append('      : "memory");')
    s.append("  }")
    s.append("};")
    return "\n".join(s) + "\n"


def generate(dmax: int = 0, aop_all: bool = True) -> str:
    out = ["// generated by paper_1709_00178_b200/gen_ring_rt.py -- do not edit\n",
           f"static_assert(PYRIT_RT_PAIR_D == {dmax} && PYRIT_RT_PAIR_AOP_ALL == {int(aop_all)}, "
           "\"ring_rt_ops.inc was generated for other PYRIT_RT_PAIR_* values\");\n"]
    for inst in instances():
        out.append(emit(*inst, dmax=dmax, aop_all=aop_all))
    return "".join(out)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    text = generate(int(argv[1]) if len(argv) > 1 else 0, bool(int(argv[2])) if len(argv) > 2 else True)
    with open(argv[0], "w") as f:
        f.write(text)


if __name__ == "__main__":
    main()

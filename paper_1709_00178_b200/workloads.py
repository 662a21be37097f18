"""The five BASELINE.json configurations as workloads (shared by bench.py and the tests).

Data: seeded synthetic bytes (counter-based mix64, identical on GPU, numpy and
the C oracle; see oracle/pyrit_oracle.c or_fill) stand in for "uniform random
bytes from seed X"; padding bytes past the unpadded fragment length are zero
(container.hpp:207-212).  Config 4's erasures {1, 6, 9, 10} are the first four
of std::shuffle(iota(0..13), mt19937_64(3)) under libstdc++ 13.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import CodeSpec, FieldSpec


@dataclass(frozen=True)
class Workload:
    cfg: int
    name: str
    op: str  # "encode" | "decode"
    fld: FieldSpec
    k: int
    m: int
    valid: int  # unpadded fragment bytes
    seed: int
    erased: tuple = field(default_factory=tuple)

    @property
    def code(self) -> CodeSpec:
        return CodeSpec(self.k, self.m, self.fld)

    @property
    def frag(self) -> int:
        """Padded fragment (symbol) size: a multiple of w * 16 bytes."""
        q = 16 * self.fld.w
        return (self.valid + q - 1) // q * q

    @property
    def strip(self) -> int:
        return self.frag // self.fld.w

    @property
    def n_out(self) -> int:
        return len(self.erased) if self.op == "decode" else self.m

    def source_bytes(self) -> int:  # BASELINE metric: source bytes (k * F)
        return self.k * self.frag

    def moved_bytes(self) -> int:  # roofline: (k + m) F encode, (k + e) F decode
        return (self.k + self.n_out) * self.frag


GF4096 = FieldSpec.aop(12)
WORKLOADS = {
    1: Workload(1, "cfg1-encode-gf16-R5-k4m2-1MiB", "encode", FieldSpec.gf16_aop(), 4, 2, 1 << 20, 0),
    2: Workload(2, "cfg2-encode-gf256-R17-k10m4-16MiB", "encode", FieldSpec.gf256_r17(), 10, 4, 16 << 20, 1),
    3: Workload(3, "cfg3-encode-gf1024-R11-k12m4-64MiB", "encode", FieldSpec.aop(10), 12, 4, 64 << 20, 2),
    4: Workload(4, "cfg4-decode-gf256-R17-k10m4-64MiB-e1,6,9,10", "decode", FieldSpec.gf256_r17(), 10, 4,
                64 << 20, 3, (1, 6, 9, 10)),
    5: Workload(5, "cfg5-encode-gf4096-R13-k16m4-512MiB", "encode", GF4096, 16, 4, 512 << 20, 4),
}


def shard(strip: int, rank: int, world: int, align: int = 16) -> tuple[int, int]:
    """Byte range [lo, hi) of every strip owned by `rank`."""
    lo = (strip * rank // world) // align * align
    hi = strip if rank == world - 1 else (strip * (rank + 1) // world) // align * align
    return lo, hi

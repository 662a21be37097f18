"""Shared test helpers: field conversions and seeded data (tests only)."""
from __future__ import annotations

import numpy as np

import oracle as O
import paper_1709_00178_b200 as P

G16 = P.FieldSpec.gf16_aop()
G64 = P.FieldSpec.gf64_esp()
G256 = P.FieldSpec.gf256_r17()
G1024 = P.FieldSpec.aop(10)
G4096 = P.FieldSpec.aop(12)


def ofield(f: P.FieldSpec) -> O.Field:
    return O.Field(f.w, f.n, f.kind, f.s, f.r_esp or f.w, f.modulus)


def rand_symbols(count: int, symbol_size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (count, symbol_size), dtype=np.uint8)


def seeded_symbols(count: int, symbol_size: int, w: int, seed: int, valid: int | None = None) -> np.ndarray:
    """Symbols built with the bench's counter-based generator (oracle.fill_np)."""
    out = np.empty((count, symbol_size), dtype=np.uint8)
    for j in range(count):
        out[j] = O.fill_np(seed, j, symbol_size, valid=valid)
    return out


def oracle_encode(f: P.FieldSpec, m: np.ndarray, data: np.ndarray, kind: int = 0) -> np.ndarray:
    """codec.hpp:444-469 restated (field oracle, column at a time)."""
    strip = data.shape[1] // f.w
    outs = O.apply_columns(ofield(f), m, [data[j] for j in range(data.shape[0])], strip, kind=kind)
    return np.stack(outs)


def oracle_ring(f: P.FieldSpec, m: np.ndarray, data: np.ndarray, kind: int = 0) -> np.ndarray:
    """schedule.hpp:94-163 + codec.hpp:118-157 restated (region ops; fast)."""
    strip = data.shape[1] // f.w
    outs = O.ring_replay(ofield(f), m, [data[j] for j in range(data.shape[0])], strip, kind=kind)
    return np.stack(outs)

"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no sums, no casts with rounding, no
block layout): it only draws per-rank gradient-like buffers, deterministic in
(kind, n, rank, seed).  Recipe:

* seed of rank r = ``seed + r`` with the default base seed 1811 (``DDL_SEED`` overrides);
  numpy PCG64.
* int32  ``uniform``   : uniform in [-2^20, 2^20).
* int32  ``bitmask``   : x_r[i] = (1 << r) | ((i mod 2^20) << 8)   (r < 8) -- a missing or
  doubled rank shows in the low byte, a misplaced element in the high bits.
* int32  ``fullrange`` : uniform over all 2^32 bit patterns (exercises two's-complement wrap).
* fp32   ``normal``    : N(0, 1).
* fp32   ``intvalued`` : integers uniform in [-2^10, 2^10) stored as fp32 (every partial sum of
  <= 2^13 ranks is exactly representable, so the sum is order-independent).
* fp32   ``rankplus1`` : x_r[i] = r + 1.
* bf16   ``normal``    : N(0, 1) drawn in fp32 and TRUNCATED to its upper 16 bits (returned as
  uint16 bit patterns).  Truncation, not the method's RNE cast, so no rounding code lives here.
* fp32 / bf16 ``specials`` : IEEE special values mixed with N(0,1): about half of the
  elements are drawn from a fixed palette of bit patterns (+-0, the smallest and largest
  subnormals, +-max finite, +-values whose pairwise sums overflow, +-inf, quiet NaNs with
  different payloads and signs), the rest are ``normal``.  Bit patterns are chosen, never
  computed, so no arithmetic of the method lives here either.
* ``resnet50`` buckets : ResNet-50's 161 parameter tensors in torch DDP's bucket order
  (resnet50_buckets.json, written by scripts/gen_resnet50_buckets.py); each tensor's values
  are N(0, (1e-2 / sqrt(fan_in))^2), the scale of a gradient at He-initialised weights.
* ``unet3d``           : 19,075,523 fp32 values N(0, 1e-3^2) as one flat buffer (SURVEY.md 8(d)
  config 3; the paper gives no parameter list).
"""
from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

BASE_SEED = int(os.environ.get("DDL_SEED", "1811"))

RESNET50_PARAMS = 25_557_032
UNET3D_PARAMS = 19_075_523


def rng(rank: int, seed: int = BASE_SEED, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed + rank, stream]))


def int32_uniform(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    return rng(rank, seed).integers(-(1 << 20), 1 << 20, size=n, dtype=np.int32)


def int32_bitmask(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    if not 0 <= rank < 8:
        raise ValueError("bitmask pattern needs rank < 8")
    i = np.arange(n, dtype=np.int64)
    return (((i % (1 << 20)) << 8) | (1 << rank)).astype(np.int32)


def int32_fullrange(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    return rng(rank, seed, 1).integers(0, 1 << 32, size=n, dtype=np.uint32).view(np.int32)


def fp32_normal(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    return rng(rank, seed, 2).standard_normal(n, dtype=np.float32)


def fp32_intvalued(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    return rng(rank, seed, 3).integers(-(1 << 10), 1 << 10, size=n).astype(np.float32)


def fp32_rankplus1(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    return np.full(n, rank + 1, dtype=np.float32)


def bf16_normal_bits(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    f = rng(rank, seed, 4).standard_normal(n, dtype=np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


# IEEE special bit patterns (SURVEY.md 8(c) ledger 9/10: no FTZ, NaNs compare equal)
FP32_SPECIALS = np.array([
    0x00000000, 0x80000000,             # +0, -0
    0x00000001, 0x80000001,             # +- smallest subnormal
    0x007FFFFF, 0x807FFFFF,             # +- largest subnormal
    0x00800000,                         # smallest normal
    0x7F7FFFFF, 0xFF7FFFFF,             # +- max finite
    0x7F160000, 0xFF160000,             # +- 2.0e38: two of them overflow
    0x7F800000, 0xFF800000,             # +- inf
    0x7FC00000, 0xFFC00001, 0x7F800001,  # NaNs: canonical, negative with payload, signalling
    0x3F800000, 0xBF800000,             # +- 1
], dtype=np.uint32)

BF16_SPECIALS = np.array([
    0x0000, 0x8000,                     # +0, -0
    0x0001, 0x8001,                     # +- smallest subnormal
    0x007F, 0x807F,                     # +- largest subnormal
    0x7F7F, 0xFF7F,                     # +- max finite
    0x7F16, 0xFF16,                     # +- 2.0e38
    0x7F80, 0xFF80,                     # +- inf
    0x7FC0, 0xFFC1, 0x7F81,             # NaNs
    0x3F80, 0xBF80,                     # +- 1
], dtype=np.uint16)


def fp32_specials(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    g = rng(rank, seed, 5)
    base = g.standard_normal(n, dtype=np.float32).view(np.uint32)
    pick = g.integers(0, len(FP32_SPECIALS), size=n)
    use = g.random(n) < 0.5
    return np.where(use, FP32_SPECIALS[pick], base).astype(np.uint32).view(np.float32)


def bf16_specials_bits(n: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    g = rng(rank, seed, 6)
    base = (g.standard_normal(n, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    pick = g.integers(0, len(BF16_SPECIALS), size=n)
    use = g.random(n) < 0.5
    return np.where(use, BF16_SPECIALS[pick], base).astype(np.uint16)


KINDS = {
    ("int32", "uniform"): int32_uniform,
    ("int32", "bitmask"): int32_bitmask,
    ("int32", "fullrange"): int32_fullrange,
    ("float32", "normal"): fp32_normal,
    ("float32", "intvalued"): fp32_intvalued,
    ("float32", "rankplus1"): fp32_rankplus1,
    ("bfloat16", "normal"): bf16_normal_bits,
    ("float32", "specials"): fp32_specials,
    ("bfloat16", "specials"): bf16_specials_bits,
}


def rank_buffers(dtype: str, kind: str, n: int, nranks: int, seed: int = BASE_SEED) -> list[np.ndarray]:
    """One buffer per rank; bf16 buffers are uint16 bit patterns."""
    f = KINDS[(dtype, kind)]
    return [f(n, r, seed) for r in range(nranks)]


@lru_cache(maxsize=1)
def resnet50_layout() -> dict:
    with open(os.path.join(os.path.dirname(__file__), "resnet50_buckets.json")) as fh:
        return json.load(fh)


def resnet50_bucket_bytes() -> list[int]:
    return [b["bytes"] for b in resnet50_layout()["buckets"]]


def resnet50_bucket(bucket: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """fp32 gradient values of one DDP bucket for one rank."""
    g = rng(rank, seed, 100 + bucket)
    parts = [g.standard_normal(t["numel"], dtype=np.float32) * np.float32(1e-2 / np.sqrt(t["fan_in"]))
             for t in resnet50_layout()["buckets"][bucket]["tensors"]]
    return np.concatenate(parts)


def unet3d_gradients(rank: int, seed: int = BASE_SEED, n: int = UNET3D_PARAMS) -> np.ndarray:
    return rng(rank, seed, 200).standard_normal(n, dtype=np.float32) * np.float32(1e-3)

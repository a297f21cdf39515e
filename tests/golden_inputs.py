"""Deterministic input recipes shared by the golden fixtures and the tests.

Values come from the reference's keyed normal01 (include/gcomm/util.hpp:32-38),
restated in numpy here so the recipes need no oracle library; edits cover
the edge cases SURVEY §4 lists (zero buckets, -0.0, spikes, ragged tails).
"""
from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    """util.hpp:14-19 vectorised over uint64 arrays."""
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01(seed, a, b):
    """util.hpp:26-29 (a, b may be arrays)."""
    seed = np.uint64(seed)
    h = mix64(seed ^ mix64(np.asarray(a, np.uint64) ^ mix64(np.asarray(b, np.uint64))))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal01(seed, idx):
    """util.hpp:32-38.  Bit-equal to the C++ for the inputs we use (glibc
    log/cos vs numpy's may differ in the last ulp of a double, which the
    float cast almost always absorbs; tests that need exact bits take inputs
    from the oracle library instead)."""
    idx = np.asarray(idx, np.uint64)
    u1 = uniform01(seed, idx, 0x6E5F)
    u2 = uniform01(seed, idx, 0x7A21)
    u1 = np.maximum(u1, 1e-300)
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)).astype(np.float32)


def make_input(n: int, gen: dict) -> np.ndarray:
    kind = gen.get("kind", "normal")
    seed = int(gen.get("seed", 0))
    scale = np.float32(gen.get("scale", 1.0))
    v = normal01(seed, np.arange(n, dtype=np.uint64)) * scale if n else np.zeros(0, np.float32)
    v = v.astype(np.float32)
    if kind == "zeros_mixed" and n:
        v[: min(n, 200)] = 0.0  # leading zero buckets
        v[n // 2: n // 2 + min(n // 4, 300)] = 0.0
    elif kind == "negzero" and n:
        v[::3] = np.float32(-0.0)
        v[1::7] = np.float32(0.0)
    elif kind == "spike" and n:
        v *= np.float32(1e-6)
        v[:: max(1, n // 5)] = np.float32(1e3)
    elif kind == "tiny_scale":
        v *= np.float32(1e-38)  # subnormal products in float, normal in double
    elif kind == "huge_scale":
        v *= np.float32(1e30)
    elif kind == "integers":
        v = np.round(8.0 * v).astype(np.float32)
    return np.ascontiguousarray(v, np.float32)

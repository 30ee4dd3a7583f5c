"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no objective, gain, screen or
ascent math): only the instance generator and
the packed-bit layout of the C-ABI (include/ubqp.h, "bit j is bit j&63 of word j>>6").
"""
from __future__ import annotations

import numpy as np

__all__ = ["generate_Q", "generate_Q_real", "pack_bits", "unpack_bits", "CONFIGS"]


def generate_Q(n: int, density: float, low: int = -100, high: int = 100, seed: int = 0) -> np.ndarray:
    """Symmetric int32 n x n instance (R2; SPEC generate_random S:58-66).

    Each unordered pair {i, j}, i <= j (diagonal included), is independently nonzero
    with probability ``density``; nonzero values are uniform integers in
    [low, high] \\ {0}.  Deterministic in (n, density, low, high, seed).
    """
    if n < 0 or not (0.0 <= density <= 1.0) or low > high:
        raise ValueError("bad generator arguments")
    vals = np.array([v for v in range(low, high + 1) if v != 0], dtype=np.int32)
    if vals.size == 0:
        raise ValueError("weight range contains only 0")
    rng = np.random.Generator(np.random.PCG64(seed))
    iu, ju = np.triu_indices(n)
    keep = rng.random(iu.shape[0]) < density
    v = vals[rng.integers(0, vals.size, size=iu.shape[0])]
    v = np.where(keep, v, 0).astype(np.int32)
    Q = np.zeros((n, n), dtype=np.int32)
    Q[iu, ju] = v
    Q[ju, iu] = v
    return Q


def generate_Q_real(n: int, density: float, low: float = -100.0, high: float = 100.0, seed: int = 0,
                    dtype=np.float64) -> np.ndarray:
    """Symmetric real instance (SURVEY Appendix B setup): pairs i <= j nonzero w.p. density,
    values uniform in [low, high)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    iu, ju = np.triu_indices(n)
    keep = rng.random(iu.shape[0]) < density
    v = np.where(keep, rng.uniform(low, high, size=iu.shape[0]), 0.0).astype(dtype)
    Q = np.zeros((n, n), dtype=dtype)
    Q[iu, ju] = v
    Q[ju, iu] = v
    return Q


def pack_bits(X: np.ndarray) -> np.ndarray:
    """uint8 0/1 [K][n] -> uint64 [K][ceil(n/64)], bit j -> bit j&63 of word j>>6; padding 0."""
    X = np.ascontiguousarray(X, dtype=np.uint8)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    K, n = X.shape
    W = (n + 63) // 64
    pad = np.zeros((K, W * 64), dtype=np.uint8)
    pad[:, :n] = X
    b = np.packbits(pad.reshape(K, W * 8, 8), axis=2, bitorder="little").reshape(K, W * 8)
    return b.view(np.uint64).reshape(K, W).copy()


def unpack_bits(B: np.ndarray, n: int) -> np.ndarray:
    """inverse of pack_bits"""
    B = np.ascontiguousarray(B, dtype=np.uint64)
    if B.ndim == 1:
        B = B.reshape(1, -1)
    K, W = B.shape
    u8 = B.view(np.uint8).reshape(K, W * 8)
    X = np.unpackbits(u8, axis=1, bitorder="little")
    return X[:, :n].copy()


# BASELINE.json configs restated concretely; seeds recorded in results.
CONFIGS = {
    1: dict(name="cfg1_n50_glover", n=50, density=0.1, seed_Q=1, K=1000, kind="glover", lam=0.5,
            max_flips=500),
    2: dict(name="cfg2_b2500_random", n=2500, density=0.1, seed_Q=2, K=1000, kind="random",
            seed_x=2),
    3: dict(name="cfg3_p5000_random", n=5000, density=1.0, seed_Q=3, K=1000, kind="random",
            seed_x=3),
    "3b": dict(name="cfg3_p7000_random", n=7000, density=1.0, seed_Q=4, K=1000, kind="random",
               seed_x=4),
    4: dict(name="cfg4_n7000_K262144_glover", n=7000, density=1.0, seed_Q=4, K=262144,
            kind="glover", lam=0.5, max_flips=70000),
}

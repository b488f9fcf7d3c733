"""Synthetic inputs: the reference's random instance generator and the
benchmark populations.

generate_urand reproduces hm/io.py:181-210 bit for bit (same SplitMix64
stream, draw order and fp64 operations), so the GPU is fed exactly the
instances the reference would build.  Host side: it runs once per instance.
"""

from __future__ import annotations

import numpy as np

from .model import Instance
from .rng import derive_stream

COORD_RANGE = 100000.0
FLOW_RANGE = 100


def euclidean_distances(coords: np.ndarray) -> np.ndarray:
    """Pairwise Euclidean distances (separate sub/mul/add/sqrt, hm/io.py:143-147)."""
    x, y = coords[:, 0], coords[:, 1]
    dx = x[:, None] - x[None, :]
    dy = y[:, None] - y[None, :]
    return np.sqrt(dx * dx + dy * dy)


def urand_coordinates(n: int, p: int, seed: int) -> np.ndarray:
    return derive_stream(seed, n, p).random_block(2 * n).reshape(n, 2) * COORD_RANGE


def generate_urand(n: int, p: int, seed: int, factors, device: bool = False) -> Instance:
    """Random Euclidean instance reproducible from (n, p, seed, factors):
    2n uniforms for x0 y0 x1 y1 ..., then n*n flows in [0, 100] row-major,
    diagonal zeroed (hm/io.py:188-210).  device=True draws and builds both
    matrices on the GPU (k_gen.cu, the same bits; n=6000 in milliseconds
    instead of seconds); the default keeps the host numpy path."""
    if n < 1:
        raise ValueError(f"node count must be positive, got {n}")
    if not 1 <= p <= n:
        raise ValueError(f"hub count p={p} outside [1, {n}]")
    chi, alpha, delta = factors
    if device:
        from ._lib import generate_urand_arrays

        dist, flow = generate_urand_arrays(n, p, seed)
        return Instance(n=n, p=p, dist=dist, flow=flow, chi=chi, alpha=alpha, delta=delta,
                        name=f"urand-n{n}-p{p}-s{seed}")
    st = derive_stream(seed, n, p)
    coords = st.random_block(2 * n).reshape(n, 2) * COORD_RANGE
    flow = st.randint_block(n * n, FLOW_RANGE + 1).astype(np.float64).reshape(n, n)
    np.fill_diagonal(flow, 0.0)
    return Instance(n=n, p=p, dist=euclidean_distances(coords), flow=flow,
                    chi=chi, alpha=alpha, delta=delta, name=f"urand-n{n}-p{p}-s{seed}")


def random_population(n: int, p: int, count: int, key: int = 1, start: int = 0) -> np.ndarray:
    """Benchmark population: individual b is the sorted set of
    the p smallest of derive_stream(key, start + b).random_block(n) (stable
    order) -- uniform p-subsets, reproducible per individual."""
    from .rng import GAMMA, _mix64_np

    out = np.empty((count, p), dtype=np.int64)
    k = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(GAMMA)
    rows = max(1, (1 << 22) // max(n, 1))
    for b0 in range(0, count, rows):
        b1 = min(count, b0 + rows)
        states = np.array([derive_stream(key, start + b).state for b in range(b0, b1)],
                          dtype=np.uint64)
        u = (_mix64_np(states[:, None] + k[None, :]) >> np.uint64(11)).astype(np.float64)
        order = np.argsort(u, axis=1, kind="stable")[:, :p]
        out[b0:b1] = np.sort(order, axis=1)
    return out

"""Seeded synthetic inputs shared by tests, bench.py and smoke() (holds none of the method's
arithmetic).

* ``sm64_np(key, k)``   -- vectorised SplitMix64 output k of the stream keyed by ``key``.
* ``uniform_vectors``   -- config-2 inputs: x[i] from sm64(seed, 2i), y[i] from sm64(seed, 2i+1);
                          fp32 = top 24 bits * 2^-24, fp64 = top 53 bits * 2^-53 (exact in both).
* ``CONFIGS``           -- the BASELINE.json configurations as parameter records.

Graph edge lists are NOT generated here: the CUDA path generates them on the device
(``nbg_graph_generate``) and the oracle generates them on the host (``oracle/orc.c``), each
implementing the same counter-based definition (reading Q9/Q11); tests compare the two
edge arrays bit for bit.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def sm64_np(key: int, k: np.ndarray) -> np.ndarray:
    k = np.asarray(k, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (k + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_vectors(n: int, seed: int, dtype=np.float32):
    """Config 2 inputs x, y ~ U[0,1) (exactly representable in dtype)."""
    idx = np.arange(n, dtype=np.uint64)
    out = []
    for off in (0, 1):
        u = sm64_np(seed, np.uint64(2) * idx + np.uint64(off))
        if dtype == np.float32:
            out.append(((u >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32))
        else:
            out.append((u >> np.uint64(11)).astype(np.float64) * 2.0**-53)
    return out[0], out[1]


# BASELINE.json configs (C1..C5) as plain records.
CONFIGS = {
    "c1": dict(graph="rmat", scale=10, edge_factor=8, dtype="fp64", alpha=0.85, itermax=20, tol=-1.0,
               dangling="uniform"),
    "c2": dict(n=1 << 24, dtypes=("fp32", "fp64")),
    "c3": dict(graph="er", scale=20, edge_factor=16, dtype="fp32", alpha=0.85, itermax=50, tol=-1.0,
               dangling="uniform"),
    "c4": dict(graph="rmat", scale=22, edge_factor=16, dtype="fp32", alpha=0.85, itermax=100, tol=1e-6,
               dangling="uniform"),
    "c5": dict(graph="rmat", scale=26, edge_factor=16, dtype="fp32", alpha=0.85, itermax=30, tol=-1.0,
               dangling="uniform"),
}

"""Counter-based candidate generator, oracle side (TEST INFRASTRUCTURE ONLY).

Reading A7/A8: the paper draws "L random initializations"
inside the per-component loop (Alg. 1; Alg. 2
"Initialize B as an L x (N-i+1) random matrix").  Entries are iid N(0,1),
fresh per component i.  The generator is bit-specified so that the oracle and
the CUDA kernel implement it independently (no shared code):

    counter  c = ((i * 2^24 + l) * 2^9 + p) * 2 + h,   p = j // 2, h in {0,1}
    z        = SplitMix64 finaliser(seed + (c + 1) * 0x9E3779B97F4A7C15 mod 2^64)
    u_h      = ((z >> 11) + 0.5) * 2^-53                  in (0, 1)
    r_{2p}   = sqrt(-2 ln u_0) cos(2 pi u_1)
    r_{2p+1} = sqrt(-2 ln u_0) sin(2 pi u_1)              (Box-Muller, fp64)

i is the 1-based component index, l the 0-based GLOBAL candidate id
(l < 2^24), j the coordinate (j < 1024).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output function (Steele, Lea, Flood 2014) on uint64 arrays."""
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniforms(seed: int, counters: np.ndarray) -> np.ndarray:
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64_mix(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * GOLDEN)
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def candidates(seed: int, i: int, ids, N: int) -> np.ndarray:
    """len(ids) x N matrix of N(0,1) draws for component i (1-based) and global ids."""
    ids = np.asarray(ids, dtype=np.uint64).reshape(-1, 1)
    P = (N + 1) // 2
    p = np.arange(P, dtype=np.uint64).reshape(1, -1)
    base = ((np.uint64(i) * np.uint64(1 << 24) + ids) * np.uint64(1 << 9) + p) * np.uint64(2)
    u0 = uniforms(seed, base)
    u1 = uniforms(seed, base + np.uint64(1))
    rad = np.sqrt(-2.0 * np.log(u0))
    out = np.empty((ids.shape[0], 2 * P), dtype=np.float64)
    out[:, 0::2] = rad * np.cos(2.0 * np.pi * u1)
    out[:, 1::2] = rad * np.sin(2.0 * np.pi * u1)
    return out[:, :N]

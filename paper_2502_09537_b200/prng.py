"""SplitMix64 (Steele, Lea & Flood), bit-compatible with dpavf/prng.py:15-60.

The reference steps a pure-Python generator one draw at a time (4*M draws
for a random state, infeasible beyond ~1e6 points).  SplitMix64's state
after k draws is seed + k*GAMMA (mod 2^64), so the stream is computed here
in one vectorised numpy pass with identical bits.
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


class SplitMix64:
    """Scalar stream (reference prng.py:15-40)."""

    def __init__(self, seed: int):
        self._state = seed & _MASK

    def next_u64(self) -> int:
        self._state = (self._state + GAMMA) & _MASK
        z = self._state
        z = ((z ^ (z >> 30)) * MIX1) & _MASK
        z = ((z ^ (z >> 27)) * MIX2) & _MASK
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))


def u64_stream(n: int, seed: int, start: int = 0) -> np.ndarray:
    """Draws start+1 .. start+n of SplitMix64(seed) as uint64."""
    k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _MASK) + k * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def uniform_array(n: int, seed: int, low: float, high: float) -> np.ndarray:
    """n deterministic uniforms in [low, high) (reference prng.py:53-60)."""
    span = high - low
    out = np.empty(n)
    chunk = 1 << 22
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        unit = (u64_stream(m, seed, s) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
        out[s:s + m] = low + span * unit
    return out

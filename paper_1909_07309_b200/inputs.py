"""Portable seeded inputs: uniform[-1,1] from a counter-based splitmix64 stream.

value_i = 2 * ((splitmix64(seed + (i+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53) - 1
(the generator of SURVEY §8(d) made counter-based so it vectorises; documented in DESIGN.md)."""
import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def uniform_pm1(n, seed, chunk=1 << 24, start=0):
    """Entries start .. start+n-1 of the seeded stream (so a rank can generate just its slab)."""
    out = np.empty(n, dtype=np.float64)
    s = np.uint64(seed)
    with np.errstate(over="ignore"):
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            z = s + (np.arange(start + lo + 1, start + hi + 1, dtype=np.uint64) * _GOLD)
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
            out[lo:hi] = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0
    return out

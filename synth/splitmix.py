"""Counter-based SplitMix64 (Steele, Lea, Flood 2014), vectorised with numpy uint64.

Element i of a stream with seed s is mix(s + (i + 1) * 0x9E3779B97F4A7C15), where
mix(z) = z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31.
Being counter-based, any element can be regenerated independently (SPEC.md S:L456 uses the
same generator for cross-language fixtures).
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 22


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Return n uint64 draws (elements offset .. offset+n-1) of the stream seeded by `seed`."""
    out = np.empty(n, dtype=np.uint64)
    s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for a in range(0, n, _CHUNK):
            b = min(n, a + _CHUNK)
            ctr = np.arange(offset + a + 1, offset + b + 1, dtype=np.uint64)
            out[a:b] = _mix(s + ctr * GOLDEN)
    return out


def uniform01(seed: int, n: int) -> np.ndarray:
    """n doubles in [0, 1) with 24 random bits each: (z >> 40) * 2^-24."""
    z = splitmix64(seed, n)
    return (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)

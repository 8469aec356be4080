"""Seeded synthetic inputs shared by the oracle side and the CUDA side of the tests and bench.

Holds none of the method's arithmetic: only the splitmix64 counter-based generator used to draw
the sampled state indices (2^20 indices uniform over [0, N), seed
0x240710925).
"""
import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n successive outputs of splitmix64 started at `seed` (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & _M64) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix64_indices(seed: int, n: int, hi: int) -> np.ndarray:
    """n indices in [0, hi): (splitmix64 output) mod hi (hi <= 2^62; the modulo bias is
    immaterial for a parity sample)."""
    return splitmix64(seed, n) % np.uint64(hi)

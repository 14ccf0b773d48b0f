import numpy as np


def rng_floats(seed: int, n: int, lo: float, hi: float, bf16_grid: bool = True) -> np.ndarray:
    """Deterministic test data (numpy PCG; the reference's own helper is
    tests/test_util.hpp:21-37)."""
    g = np.random.default_rng(seed)
    x = (lo + (hi - lo) * g.random(n)).astype(np.float32)
    if bf16_grid:
        x = bf16_grid_round(x)
    return x


def bf16_grid_round(x: np.ndarray) -> np.ndarray:
    """RNE to the bf16 grid (same rule as src/numerics.cpp:237-243)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    out = b.astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    out[nan] = x[nan]
    return out

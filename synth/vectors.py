"""Seeded test vectors (PCG64), shared by both sides. No method arithmetic."""
import numpy as np


def seeded_normal(n: int, seed: int = 7) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(n)

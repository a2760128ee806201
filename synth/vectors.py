"""Seeded test vectors: x_i = U(-1,1) + i U(-1,1) (BASELINE.json configs[0])."""
import numpy as np


def seeded_vector(n, seed):
    rng = np.random.default_rng(seed)
    re = rng.uniform(-1.0, 1.0, n)
    im = rng.uniform(-1.0, 1.0, n)
    return re + 1j * im

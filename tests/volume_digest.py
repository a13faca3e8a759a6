"""Seeded projection vectors of the volume-field digest (shared by
tools/make_volume_goldens.py, which records the reference's projections,
and the GPU test, which recomputes them for the device field)."""

import numpy as np

N_PROJ = 16


def projections(shape, n=N_PROJ, seed=77):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(shape) + 1j * rng.standard_normal(shape) for _ in range(n)]

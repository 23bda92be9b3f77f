"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds input production ONLY: no SPH arithmetic (no kernel, no
density, no force, no neighbour search). Both `oracle/` and the CUDA path
consume what it generates; neither imports the other.
"""
from .generators import (  # noqa: F401
    Particles, CONFIGS, make, c1, c2, c2_exact, fcc_exact, c3, c4, c4_weak, c5, tiny,
    quantise_positions, subsample_box, edges_unquantised,
)

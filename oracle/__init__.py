"""fp64 CPU oracle for the SPH hot path of Gonnet, "Efficient and scalable
algorithms for smoothed particle hydrodynamics on hybrid shared/distributed-
memory architectures" (arXiv:1404.2303).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this package.
The product path (`paper_1404_2303_b200`) never imports it and shares no code
with it; the only common dependency is the input generator package
`workloads/`, which holds no SPH arithmetic.

Citations: `P:<line>` = /root/reference/PAPER.md line (section / equation named
beside it); readings R1..R23 are SURVEY.md §8(c), restated in DESIGN.md.

Form: plain definitions, gather form (each target particle sums over its own
neighbours), fp64 throughout, inputs are the fp32 arrays promoted exactly.
Neighbour search uses scipy's cKDTree (a library primitive, pinned against
brute force in tests/test_oracle_neighbours.py).

Parity status per function:
  kernel.*            pinned: closed-form values, normalisation, FD derivatives
  neighbours.*        pinned: brute force on tiny periodic inputs
  sph.n_ngb_of_h      pinned: lattice closed forms, FD, monotonicity
  sph.solve_h         pinned: lattice closed forms h/Delta, root property
  sph.density_at      pinned: isolated particle, lattice rho/Omega/n_nbr closed
                      forms, Omega identity, linear-velocity div/curl closed forms
  sph.particle_state  pinned: via force pins (two-particle hand derivation)
  sph.force_at        pinned: lattice zero force, two-particle hand derivation,
                      momentum/energy conservation, viscous heating >= 0
"""
from . import kernel, neighbours, sph  # noqa: F401
from .sph import (  # noqa: F401
    OracleConfig, n_ngb_of_h, solve_h, density_at, particle_state, force_at,
    evaluate_all,
)

"""Velocity-Verlet (kick-drift-kick) time stepping around the hot path (SURVEY 8(f) f1,
first part; "integrated using a velocity-Verlet integrator") with the global
time step of Eq. 6 (C_CFL = 1/4 as in P:1353). Every arithmetic step runs in
libsph (sph_kick, sph_drift, sph_timestep, and the three hot-path calls); this class holds
the device arrays and the order of the calls. Each step rebuilds the cells from the moved
positions (or reuses them) and warm-starts h from the previous step (the regime SURVEY
8(d) calls warm).
Each step keeps the cells of the last full sort while the particles moved little
(sph_update_cells, the pseudo-Verlet reuse of P:1281-1289). Not here yet: the multiple
time-stepping integrator (the library side is sph_set_active)."""
from __future__ import annotations

from .sph import Context


class Leapfrog:
    def __init__(self, ctx: Context, x, v, m, u, c_cfl: float = 0.25):
        """x, v, m, u: contiguous float32 CUDA tensors (copied; the caller's stay untouched)."""
        self.ctx, self.c_cfl = ctx, c_cfl
        self.x, self.v, self.m, self.u = x.clone(), v.clone(), m.clone(), u.clone()
        self.h = None
        self._evaluate(None)

    def _evaluate(self, h0, v=None, u=None):
        ctx = self.ctx
        v = self.v if v is None else v
        u = self.u if u is None else u
        if h0 is None:
            ctx.build_cells(self.x, None)
        else:                                 # pseudo-Verlet: the cells are kept while they are valid
            ctx.update_cells(self.x, h0)
        d = ctx.density(v, self.m, u)
        f = ctx.force(v)
        self.h, self.rho, self.a, self.dudt, self.vsig = d.h, d.rho, f.a, f.dudt, f.vsig
        self.stats_density, self.stats_force = d.stats, f.stats

    def timestep(self) -> float:
        return self.ctx.timestep(self.h, self.vsig, self.c_cfl)

    def step(self, dt: float | None = None) -> float:
        """One KDK step of size dt (default: Eq. 6 from the current state)."""
        dt = self.timestep() if dt is None else dt
        ctx = self.ctx
        ctx.kick(self.v, self.a, 0.5 * dt, self.u, self.dudt)
        ctx.drift(self.x, self.v, dt)
        # the loops see v and u predicted to the end of the step (v and u enter the viscosity,
        # P and c; with the half-step values the energy error would be first order in dt)
        vp, up = self.v.clone(), self.u.clone()
        ctx.kick(vp, self.a, 0.5 * dt, up, self.dudt)
        self._evaluate(self.h, vp, up)        # warm start: h of the previous step
        ctx.kick(self.v, self.a, 0.5 * dt, self.u, self.dudt)
        return dt

    # diagnostics (reductions for tests and reports, not part of the step)
    def momentum(self):
        return (self.m[:, None].double() * self.v.double()).sum(0)

    def energy(self) -> float:
        m, v, u = self.m.double(), self.v.double(), self.u.double()
        return float((0.5 * m * (v * v).sum(1) + m * u).sum())

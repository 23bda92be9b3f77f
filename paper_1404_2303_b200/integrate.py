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


class MultiStep:
    """Individual power-of-two time steps (as in Gadget-2): particle i moves
    with a step 2^k dt_min <= its Eq. 6 step, kick-drift-kick per particle; at each
    synchronisation point only the particles whose step ends there are the targets of the
    density and force loops (sph_set_active), the others stay sources with their last state.
    The loops see every particle's v and u predicted to the current time. Limiter (Saitoh &
    Makino style): a step grows at most 2x at a time, and a particle whose step exceeds 4x a
    force neighbour's new step is woken (sph_neighbour_min), its step ending early."""

    def __init__(self, ctx: Context, x, v, m, u, dt_max: float, n_bins: int = 6, c_cfl: float = 0.25,
                 limiter: bool = True):
        import torch
        self.ctx, self.c_cfl, self.n_bins, self.limiter = ctx, c_cfl, n_bins, limiter
        self.dt_min = dt_max / (1 << n_bins)
        self.x, self.v, self.m, self.u = x.clone(), v.clone(), m.clone(), u.clone()
        n = x.shape[0]
        dev = x.device
        self.h = torch.empty(n, device=dev)
        self.rho = torch.empty(n, device=dev)
        self.a = torch.empty(n, 3, device=dev)
        self.dudt = torch.empty(n, device=dev)
        self.vsig = torch.empty(n, device=dev)
        self.ti = 0
        self.ti_begin = torch.zeros(n, dtype=torch.int64, device=dev)
        ctx.set_active(None)
        ctx.build_cells(self.x, None)
        ctx.density(self.v, self.m, self.u, out=dict(h=self.h, rho=self.rho))
        ctx.force(self.v, out=dict(a=self.a, dudt=self.dudt, vsig=self.vsig))
        self.step_ticks = self._ticks(None, 0)
        self._kick(self.step_ticks.float() * 0.5 * self.dt_min)
        self.evaluations = n

    def _ticks(self, sel, ti, cap2=False):
        """Power-of-two step (in dt_min ticks) <= the Eq. 6 step, dividing ti, for the particles
        in `sel` (the others keep theirs); at most 2x the previous one with cap2 (libsph
        sph_timebins)."""
        old = getattr(self, "step_ticks", None)
        return self.ctx.timebins(self.h, self.vsig, self.c_cfl, self.dt_min, self.n_bins, ti,
                                 active=sel if old is not None else None, ticks_in=old, cap2=cap2)

    def _kick(self, dt):
        self.ctx.kick_each(self.v, self.a, dt.float().contiguous(), self.u, self.dudt)

    def step(self) -> float:
        import torch
        ctx = self.ctx
        end = self.ti_begin + self.step_ticks
        ti_end = int(end.min())
        dt = (ti_end - self.ti) * self.dt_min
        ctx.drift(self.x, self.v, dt)
        active = end == ti_end
        # v and u predicted to ti_end: v holds the mid-step value of each particle's step
        pred = ((ti_end - (self.ti_begin + self.step_ticks // 2)).float() * self.dt_min).contiguous()
        vp, up = self.v.clone(), self.u.clone()
        ctx.kick_each(vp, self.a, pred, up, self.dudt)
        ctx.set_active(active)
        ctx.update_cells(self.x, self.h)
        ctx.density(vp, self.m, up, out=dict(h=self.h, rho=self.rho))
        ctx.force(vp, out=dict(a=self.a, dudt=self.dudt, vsig=self.vsig))
        self.evaluations += int(active.sum())
        zero = torch.zeros_like(self.h)
        self._kick(torch.where(active, self.step_ticks.float() * 0.5 * self.dt_min, zero))   # close the step
        # a step grows at most 2x at a time (the limiter) ...
        self.step_ticks = self._ticks(active, ti_end, cap2=self.limiter)
        if self.limiter:
            # ... and no particle keeps a step above 4x a force neighbour's new one: such a
            # particle is woken, its current step ending at the next point of the shorter grid
            # (never later than its current end), its opening half kick corrected (libsph
            # sph_neighbour_min + sph_timebins_wake)
            lim = torch.full_like(self.h, float("inf"))
            ctx.neighbour_min(torch.where(active, self.step_ticks.float(), torch.full_like(self.h, float("inf"))), lim)
            self._kick(ctx.timebins_wake(active, lim, ti_end, self.ti_begin, self.step_ticks, self.dt_min))
        self._kick(torch.where(active, self.step_ticks.float() * 0.5 * self.dt_min, zero))   # open the next
        self.ti_begin = torch.where(active, torch.full_like(self.ti_begin, ti_end), self.ti_begin)
        self.ti = ti_end
        return dt

    def time(self) -> float:
        return self.ti * self.dt_min

    def synced_energy(self) -> float:
        """Total energy at the current time when every particle starts a step here."""
        import torch
        assert bool((self.ti_begin == self.ti).all()), "not a synchronisation point"
        half = (self.step_ticks.float() * 0.5 * self.dt_min)[:, None]
        v = self.v.double() - self.a.double() * half.double()
        u = self.u.double() - self.dudt.double() * half[:, 0].double()
        m = self.m.double()
        return float((0.5 * m * (v * v).sum(1) + m * u).sum())

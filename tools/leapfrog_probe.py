"""Energy / momentum drift of the velocity-Verlet loop vs C_CFL (order check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
from paper_1404_2303_b200.integrate import Leapfrog
p = workloads.tiny(11, n=4000, clump_frac=0.3, n_dup=0)
t = lambda q: torch.from_numpy(np.ascontiguousarray(q)).cuda()
for name, cfg in [("tiny", p), ("c1", workloads.c1())]:
    for c in [0.25, 0.1, 0.05, 0.025]:
        ctx = sph.Context(sph.default_config(cfg.box, n_ngb_tol=1e-4, split_count=48, split_fraction=0.0))
        lf = Leapfrog(ctx, t(cfg.x), t(cfg.v), t(cfg.m), t(cfg.u), c_cfl=c)
        E0 = lf.energy(); P0 = lf.momentum()
        T = 0.0; steps = 0
        dt0 = lf.timestep()
        Tend = 20 * 0.25 / c * dt0 if c == 0.25 else Tend
        while T < Tend and steps < 2000:
            T += lf.step(min(lf.timestep(), Tend - T + 1e-12)); steps += 1
        print(name, "cfl", c, "steps", steps, "T", T, "dE/E", (lf.energy() - E0) / E0, "dP", float((lf.momentum() - P0).abs().max()))
        ctx.close()

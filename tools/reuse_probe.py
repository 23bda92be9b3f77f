"""Warm C4 step with a full build vs with the kept cells (sph_update_cells) after a small drift."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
p = workloads.make("C4")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
ctx = sph.Context(sph.default_config(p.box, split_count=48, split_fraction=0.0))
ctx.build_cells(x); h = ctx.density(v, m, u).h.clone(); ctx.force(v)
rng = np.random.default_rng(1)
x2 = t(np.mod(p.x + rng.uniform(-1, 1, p.x.shape).astype(np.float32) * 0.02 * float(h.min()), 1.0).astype(np.float32))
for mode in ["full", "reuse", "full", "reuse"]:
    best = 1e9
    for _ in range(4):
        if mode == "reuse":
            ctx.build_cells(x, h); ctx.density(v, m, u); ctx.force(v)
        torch.cuda.synchronize()
        if mode == "full":
            ctx.build_cells(x2, h)
        else:
            ctx.update_cells(x2, h)
        d = ctx.density(v, m, u); f = ctx.force(v)
        tot = d.stats["ms_build"] + d.stats["ms_density"] + f.stats["ms_force"]
        best = min(best, tot)
    print(mode, "ms %.2f" % best, "build %.2f" % d.stats["ms_build"], "reused", d.stats["cells_reused"])

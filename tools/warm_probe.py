"""Warm-start timing (h0 = converged h x (1 + 0.05 U(-1,1))) for a few h_margin values."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_2303_b200 as sph, workloads
p = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, v, m, u = t(p.x), t(p.v), t(p.m), t(p.u)
base = dict(split_count=48, split_fraction=0.0)
ctx = sph.Context(sph.default_config(p.box, **base))
ctx.build_cells(x, None)
h = ctx.density(v, m, u).h.clone()
ctx.close()
rng = np.random.default_rng(140423099)
h0 = (h * t((1 + 0.05 * rng.uniform(-1, 1, p.n)).astype(np.float32))).contiguous()
for hm in [1.0, 1.03, 1.05, 1.1, 1.15]:
    ctx = sph.Context(sph.default_config(p.box, h_margin=hm, **base))
    best = None
    for _ in range(4):
        ctx.build_cells(x, h0)
        d = ctx.density(v, m, u)
        f = ctx.force(v)
        torch.cuda.synchronize()
        tot = d.stats["ms_build"] + d.stats["ms_density"] + f.stats["ms_force"]
        best = tot if best is None else min(best, tot)
    print(json.dumps({"h_margin": hm, "ms_step": best, "h_iters": d.stats["h_iters"]}), flush=True)
    ctx.close()
